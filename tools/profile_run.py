"""One propagation of a bench workload, for ncu captures (no timing)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2506_13241_b200 as pp  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "config1"]
circ = bench.build_circuit(pp, wl)
n, site, eps = wl[1], wl[4], wl[5]
init = np.zeros((1, 4), np.uint64)
init[0, site // 32] = np.uint64(3) << np.uint64(2 * (site % 32))
eng = pp.Engine(n, eps)
eng.set_initial(init, np.array([1.0]))
rows = eng.run_circuit(circ)
print(rows[-1])
