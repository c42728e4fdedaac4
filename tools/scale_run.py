"""Large single-GPU propagation with per-layer timing and property checks
(norm conservation at epsilon0 = 0).  Usage:
  python tools/scale_run.py config0_t10"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2506_13241_b200 as pp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config0_t10"
wl = bench.WORKLOADS[name]
circ = bench.build_circuit(pp, wl)
n, site, eps = wl[1], wl[4], wl[5]
init = np.zeros((1, 4), np.uint64)
init[0, site // 32] = np.uint64(3) << np.uint64(2 * (site % 32))
eng = pp.Engine(n, eps)
eng.set_initial(init, np.array([1.0]))
L = circ.num_layers()
rows = []
for t in range(1, L + 1):
    layer = circ.layers[L - t]
    sg = 0
    t0 = time.perf_counter()
    eng.apply_gates(list(reversed(layer)))
    dt = time.perf_counter() - t0
    row = {"t": t, "term_count": eng.term_count(), "observable": eng.expectation_zero_state(), "seconds": dt}
    if eps == 0.0:
        row["norm2"] = eng.norm2()
    rows.append(row)
    print(json.dumps(row), flush=True)
