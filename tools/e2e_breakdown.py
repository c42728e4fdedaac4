"""Where the e2e (simulate()) time goes: engine creation, set_initial,
run_circuit, for fresh engines vs one reused engine."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_13241_b200 as pp  # noqa: E402

wl = bench.WORKLOADS["config1"]
circ = bench.build_circuit(pp, wl)
init = np.zeros((1, 4), np.uint64)
init[0, 62 // 32] = np.uint64(3) << np.uint64(2 * (62 % 32))
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e = pp.Engine(127, 0.0)
    t1 = time.perf_counter()
    e.set_initial(init, np.array([1.0]))
    t2 = time.perf_counter()
    e.run_circuit(circ)
    t3 = time.perf_counter()
    del e
    t4 = time.perf_counter()
    out = pp.simulate(circ, observable="Z62", epsilon0=0.0)
    t5 = time.perf_counter()
    print(f"fresh: create {1e3*(t1-t0):.3f} set_initial {1e3*(t2-t1):.3f} run {1e3*(t3-t2):.3f} destroy {1e3*(t4-t3):.3f} simulate {1e3*(t5-t4):.3f} ms")
e = pp.Engine(127, 0.0)
for rep in range(4):
    t1 = time.perf_counter()
    e.set_initial(init, np.array([1.0]))
    t2 = time.perf_counter()
    e.run_circuit(circ)
    t3 = time.perf_counter()
    print(f"reused: set_initial {1e3*(t2-t1):.3f} run {1e3*(t3-t2):.3f} ms")
