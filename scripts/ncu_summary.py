"""Summarise an `ncu --set full` capture of one config's NCS step (one launch
of each kernel) into the committed profile files:

  profiles/<round>_ncu_<cfg>.csv   key metrics per kernel
  profiles/ncu_<cfg>.json          per-launch DRAM bytes, L2 hit rate,
                                   shared-memory wavefront share, issue-active
                                   share and instructions per kernel, keyed by
                                   bench.py's phase names (read by bench.py's
                                   per-kernel roofline table)

usage: python scripts/ncu_summary.py gpurun_out/x.ncu-rep <round> <cfg>
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_shared_mem"]
# bench.py phase names of the step's kernels
ALIAS = {"bp_gather_kernel": "adjoint", "bp_tile_kernel": "adjoint", "fp_orbit_kernel": "forward",
         "fp_strip_kernel": "forward", "fft_rows_r2c_kernel": "fft_rows_r2c",
         "fft_cols_filter_kernel": "fft_cols", "fft_rows_c2r_kernel": "fft_rows_c2r",
         "make_quad_kernel": "make_quad", "dual_update_kernel": "dual_update",
         "fft_rows_r2c_p2": "fft_rows_r2c", "fft_cols_filter_p2": "fft_cols",
         "fft_rows_c2r_p2": "fft_rows_c2r"}


def short(name: str) -> str:
    return name.split("(")[0].split("<")[0].split("::")[-1].strip()


def num(v: str) -> float:
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return float("nan")


def to_bytes(v: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return num(v) * scale


def main(rep: str, rnd: str, cfg: str) -> None:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    col = {k: h.index(k) for k in KEYS if k in h}
    seen = {}
    for r in rows[2:]:
        k = short(r[h.index("Kernel Name")])
        seen.setdefault(k, r)  # first launch of each kernel
    with open(f"profiles/{rnd}_ncu_{cfg}.csv", "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["Kernel Name"] + KEYS)
        w.writerow([""] + [units[col[k]] if k in col else "" for k in KEYS])
        for k, r in seen.items():
            w.writerow([k] + [r[col[m]] if m in col else "" for m in KEYS])
    summ = {"source": f"profiles/{rnd}_ncu_{cfg}.csv (ncu --set full --clock-control none, "
                      f"one launch of each kernel, config {cfg})", "kernels": {}}
    for k, r in seen.items():
        name = ALIAS.get(k, k)

        def get(m, _r=r):
            return num(_r[col[m]]) if m in col else None

        rd = to_bytes(r[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]])
        wr = to_bytes(r[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]])
        du = units[col["gpu__time_duration.sum"]]
        dur = get("gpu__time_duration.sum") * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(du, 1.0)
        wf = get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")
        ia = get("smsp__issue_active.avg.pct_of_peak_sustained_active")
        hr = get("lts__t_sector_hit_rate.pct")
        summ["kernels"][name] = {
            "kernel": k, "duration_us": dur, "dram_bytes": rd + wr,
            "l2_hit_rate": None if hr is None else hr / 100,
            "dram_gbs": (rd + wr) / (dur * 1e-6) / 1e9 if dur else None,
            "smem_wavefront_frac": None if wf is None else wf / 100,
            "issue_active_frac": None if ia is None else ia / 100,
            "inst_per_launch": get("smsp__inst_executed.sum"),
            "smem_wavefronts": get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "smem_bank_conflicts": get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "grid": get("launch__grid_size"), "registers": get("launch__registers_per_thread")}
    with open(f"profiles/ncu_{cfg}.json", "w") as fh:
        json.dump(summ, fh, indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "r2",
         sys.argv[3] if len(sys.argv) > 3 else "c3")
