"""One propagation of a bench workload, for ncu captures (no timing).

usage: profile_run.py <workload> [--warm]
--warm runs the propagation once untimed on the same engine, then brackets
the second (steady-state: arenas sized, graphs captured) with
cudaProfilerStart/Stop, for `ncu --profile-from-start off`.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2506_13241_b200 as pp  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
warm = "--warm" in sys.argv
wl = bench.WORKLOADS[args[0] if args else "config1"]
circ = bench.build_circuit(pp, wl)
n, site, eps = wl[1], wl[4], wl[5]
init = np.zeros((1, 4), np.uint64)
init[0, site // 32] = np.uint64(3) << np.uint64(2 * (site % 32))
eng = pp.Engine(n, eps)
if warm:
    import torch
    eng.set_initial(init, np.array([1.0]))
    eng.run_circuit(circ)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
t0 = time.perf_counter()
eng.set_initial(init, np.array([1.0]))
rows = eng.run_circuit(circ)
t1 = time.perf_counter()
if warm:
    torch.cuda.profiler.stop()
print(rows[-1], f"host wall {1e3 * (t1 - t0):.3f} ms")
