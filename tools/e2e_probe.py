import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["NMFA_TIMING"] = "1"
import numpy as np, torch
import paper_1806_08422_b200 as nb
from paper_1806_08422_b200 import _native
p = nb.gen_sk(2000, 7)
temps = nb.DEFAULT_SCHEDULE.temperatures(1000)
R = 8192
cfg = torch.empty((R, 2000), dtype=torch.int8).pin_memory()
en = torch.empty(R, dtype=torch.float64).pin_memory()
lib = _native.load()
h = p.device_handle().handle
for k in range(4):
    t0 = time.perf_counter()
    _native.check(lib.nmfa_anneal_host(h, R, 1000, _native.ptr(temps), 0.15, 0.15, k, 0, _native.ptr(cfg), _native.ptr(en)))
    print(f"call {k}: {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
