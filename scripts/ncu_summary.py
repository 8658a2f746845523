"""Summarise an `ncu --set full` capture of the C3 step (one launch of each
kernel) into the committed profile files:

  profiles/<round>_ncu_kernels.csv  key metrics per kernel
  profiles/ncu_traffic.json         per-launch DRAM bytes, shared-memory
                                    wavefront share, issue-active share and
                                    instructions (read by bench.py's roofline)

usage: python scripts/ncu_summary.py gpurun_out/x.ncu-rep r1
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_shared_mem"]
# bench.py phase names of the two projector kernels
ALIAS = {"bp_gather_kernel": "adjoint", "bp_tile_kernel": "adjoint", "fp_orbit_kernel": "forward",
         "fp_strip_kernel": "forward"}


def short(name: str) -> str:
    base = name.split("(")[0].split("<")[0].split("::")[-1].strip()
    return base


def to_bytes(v: str, unit: str) -> float:
    f = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return f * scale


def main(rep: str, rnd: str) -> None:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    seen = {}
    for r in rows[2:]:
        k = short(r[h.index("Kernel Name")])
        seen.setdefault(k, r)  # first launch of each kernel
    with open(f"profiles/{rnd}_ncu_kernels.csv", "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["Kernel Name"] + KEYS)
        w.writerow([""] + [units[h.index(k)] if k in h else "" for k in KEYS])
        for k, r in seen.items():
            w.writerow([k] + [r[h.index(m)] if m in h else "" for m in KEYS])
    summ = {"source": f"profiles/{rnd}_ncu_kernels.csv (ncu --set full, one launch each, C3)",
            "dram_bytes_per_launch": {}, "smem_wavefront_frac": {}, "issue_active_frac": {},
            "inst_per_launch": {}, "duration_us": {}}
    for k, r in seen.items():
        name = ALIAS.get(k, k)
        rd = to_bytes(r[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_read.sum")])
        wr = to_bytes(r[h.index("dram__bytes_write.sum")], units[h.index("dram__bytes_write.sum")])
        summ["dram_bytes_per_launch"][name] = rd + wr
        m = "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"
        summ["smem_wavefront_frac"][name] = float(r[h.index(m)]) / 100
        m = "smsp__issue_active.avg.pct_of_peak_sustained_active"
        summ["issue_active_frac"][name] = float(r[h.index(m)]) / 100
        summ["inst_per_launch"][name] = float(r[h.index("smsp__inst_executed.sum")].replace(",", ""))
        du = units[h.index("gpu__time_duration.sum")]
        summ["duration_us"][name] = float(r[h.index("gpu__time_duration.sum")].replace(",", "")) * {
            "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(du, 1.0)
    with open("profiles/ncu_traffic.json", "w") as fh:
        json.dump(summ, fh, indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "r1")
