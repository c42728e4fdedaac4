"""Heavy-hex kicked Ising at eps0 > 0 (BASELINE config 2 shape): propagate
layers 1..t-1 untimed, then bracket layer t with cudaProfilerStart/Stop (for
`ncu --profile-from-start off`) and print per-layer wall time, |O| and the
engine's trace.  No bench numbers come from here.

  python tools/eps_profile.py --theta 0.25 --eps 2e-5 --t 10
"""
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
ap.add_argument("--eps", type=float, default=2e-5)
ap.add_argument("--t", type=int, default=10)
args = ap.parse_args()

import torch  # noqa: E402

one = pp.build_kicked_ising(pp.heavy_hex_127(), f"{args.theta!r}pi", "-0.5pi", 1)
eng = pp.Engine(127, args.eps)
z62 = np.asarray(pp.parse_pauli_label("Z62", 127).words, np.uint64)[None]
eng.set_initial(z62, np.array([1.0]))
for t in range(1, args.t + 1):
    torch.cuda.synchronize()
    if t == args.t:
        eng.kernel_stats()
        torch.cuda.profiler.start()
    t0 = time.perf_counter()
    row = eng.run_circuit(one)[0]
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if t == args.t:
        torch.cuda.profiler.stop()
        ks = eng.kernel_stats()
    print(json.dumps({"t": t, "term_count": row["term_count"], "observable": row["observable"], "seconds": dt}),
          flush=True)
print(json.dumps({"kernel_stats_last_layer": ks}), flush=True)
g, st = eng.group_sizes()
print(json.dumps({"group_sizes_log2": {b: [g[b], st[b]] for b in range(64) if g[b]}}), flush=True)
