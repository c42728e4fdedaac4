"""BASELINE config 2 on one GPU: heavy-hex kicked Ising, Z62, 20 steps,
theta_h in pi units, per-gate truncation at a given epsilon0.  Prints one
JSON row per layer (|O|, <Z62>, device seconds) and a summary with the peak
|O| and string-gates/s (string-gates counted from per-gate |O_in| when
--count is given, in a separate untimed run).

  python tools/config2_sweep.py --theta 0.25 --eps 1e-5 [--steps 20] [--count]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2506_13241_b200 as pp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--theta", type=float, default=0.25, help="theta_h in units of pi")
ap.add_argument("--eps", type=float, default=1e-5)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--max-terms", type=float, default=2.0e9)
ap.add_argument("--count", action="store_true")
args = ap.parse_args()

circ = pp.build_kicked_ising(pp.heavy_hex_127(), f"{args.theta!r}pi", "-0.5pi", args.steps)
z62 = np.asarray(pp.parse_pauli_label("Z62", 127).words, np.uint64)[None]
L = circ.num_layers()


def run(count):
    eng = pp.Engine(127, args.eps, "gate", max_terms=int(args.max_terms))
    eng.set_initial(z62, [1.0])
    rows, sg, peak = [], 0, 1
    t_all = time.perf_counter()
    for t in range(1, L + 1):
        layer = list(reversed(circ.layers[L - t]))
        t0 = time.perf_counter()
        try:
            if count:
                for g in layer:
                    sg += eng.term_count()
                    eng.apply_gate(g)
                    peak = max(peak, eng.term_count())
            else:
                eng.apply_gates(layer)
        except pp.ResourceLimitError as exc:
            rows.append({"t": t, "resource_limit": str(exc)})
            print(json.dumps(rows[-1]), flush=True)
            break
        dt = time.perf_counter() - t0
        row = {"t": t, "term_count": eng.term_count(), "observable": eng.expectation_zero_state(), "seconds": dt}
        peak = max(peak, row["term_count"])
        rows.append(row)
        print(json.dumps(row), flush=True)
    return rows, sg, peak, time.perf_counter() - t_all


rows, _, peak, total = run(False)
out = {"theta_h_pi": args.theta, "epsilon0": args.eps, "steps": args.steps, "peak_terms_layer_end": peak,
       "seconds": total, "final": rows[-1]}
if args.count:
    crow, sg, cpeak, _ = run(True)
    out.update({"string_gates": sg, "peak_terms": cpeak, "string_gates_per_s": sg / total})
print(json.dumps({"summary": out}), flush=True)
