"""Worker start-up cost split: numpy import, libest load, CUDA context, worker
modules, first allocation (the per-process part of the rescale restart stage)."""
import time, sys
t0 = time.perf_counter()
sys.path.insert(0, '.')
import numpy
t1 = time.perf_counter()
from paper_2512_19851_b200.device import Device
t2 = time.perf_counter()
d = Device(0)
t3 = time.perf_counter()
import paper_2512_19851_b200.worker, paper_2512_19851_b200.ipc, paper_2512_19851_b200.executor
t4 = time.perf_counter()
p = d.alloc(1 << 20); d.sync()
t5 = time.perf_counter()
print(f"numpy {1e3*(t1-t0):.0f} ms, libest import {1e3*(t2-t1):.0f} ms, ctx {1e3*(t3-t2):.0f} ms, worker modules {1e3*(t4-t3):.0f} ms, first alloc {1e3*(t5-t4):.0f} ms")
