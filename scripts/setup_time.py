import sys, time
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1810_13100_b200 import configs, instances, ncsg
cfg = configs.get('c3')
mask = instances.metric_mask(cfg)
b = np.zeros((cfg.angles, cfg.det))
ncsg.lib()
for rep in range(3):
    t = time.perf_counter(); r = ncsg.RadonMap(cfg.n, cfg.angles, cfg.det); t1 = time.perf_counter() - t
    t = time.perf_counter(); p = ncsg.ct_problem(cfg, b, mask=mask); t2 = time.perf_counter() - t
    t = time.perf_counter(); p.set_state(); p.step(1); p.sync(); t3 = time.perf_counter() - t
    t = time.perf_counter(); res = p.solve(1000, record_every=1000); t4 = time.perf_counter() - t
    print(f'radon {t1*1e3:.1f} ms  problem {t2*1e3:.1f} ms  first step {t3*1e3:.1f} ms  solve1000 {t4*1e3:.1f} ms')
    del r, p
