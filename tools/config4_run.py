"""BASELINE config 4 shape on one GPU: non-Clifford kicked Ising on the
127-qubit heavy-hex lattice (theta_J = -pi/2 + 0.2, so Rzz branches too),
theta_h = 0.4, O0 = sum_i Z_i / 127, per-gate truncation at epsilon0.
Prints one JSON row per layer and a summary.

  python tools/config4_run.py --eps 1e-4 --steps 12"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2506_13241_b200 as pp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--eps", type=float, default=1e-4)
ap.add_argument("--steps", type=int, default=12)
ap.add_argument("--max-terms", type=float, default=0)
args = ap.parse_args()

circ = pp.build_kicked_ising(pp.heavy_hex_127(), 0.4, -math.pi / 2 + 0.2, args.steps)
words = np.stack([np.asarray(pp.parse_pauli_label(f"Z{q}", 127).words, np.uint64) for q in range(127)])
eng = pp.Engine(127, args.eps, "gate", max_terms=int(args.max_terms))
eng.set_initial(words, np.full(127, 1.0 / 127))
L = circ.num_layers()
t_all = time.perf_counter()
peak = 0
for t in range(1, L + 1):
    t0 = time.perf_counter()
    eng.apply_gates(list(reversed(circ.layers[L - t])))
    row = {"t": t, "term_count": eng.term_count(), "observable": eng.expectation_zero_state(),
           "seconds": time.perf_counter() - t0}
    peak = max(peak, row["term_count"])
    print(json.dumps(row), flush=True)
print(json.dumps({"summary": {"epsilon0": args.eps, "steps": L, "peak_terms_layer_end": peak,
                              "seconds": time.perf_counter() - t_all}}), flush=True)
