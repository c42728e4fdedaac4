"""Shape of the work the dense Rx sublayer sees at BASELINE config 0, t = 10:
propagate 9 layers, apply layer 10's ZZ run only, export, and histogram the
z-groups by m = popcount(z) (the stage count) and by input size.  Diagnostic
only (prints JSON)."""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2506_13241_b200 as pp  # noqa: E402

geom = pp.load_geometry("\n".join(f"{i} {i + 1} {i % 2}" for i in range(63)))
circ = pp.build_kicked_ising(geom, 0.3, "-0.5pi", 9)
eng = pp.Engine(64, 0.0)
eng.set_initial(O.site_word(32, 3)[None], np.array([1.0]))
eng.run_circuit(circ)
layer = list(circ.layers[0])
zz = [g for g in reversed(layer) if g.cos_theta == 0.0]
eng.apply_gates(zz)
w, c = eng.export()
x, z = O.to_planes(w)
z = z[:, 0] if z.ndim == 2 else z
zu, inv, cnt = np.unique(z, return_inverse=True, return_counts=True)
x = x[:, 0] if x.ndim == 2 else x
F = x & ~z
pairs = np.unique(np.stack([z, F], 1), axis=0)
pz, pcls = np.unique(pairs[:, 0], return_counts=True)  # classes per z-group (same order as zu)
m = np.array([bin(int(v)).count("1") for v in zu])
out = {"strings": int(len(c)), "groups": int(len(zu)), "classes": int(len(pairs))}
by_m = collections.defaultdict(lambda: [0, 0, 0, 0])
for mm, cc, kk in zip(m, cnt, pcls):
    e = by_m[int(mm)]
    e[0] += 1
    e[1] += int(cc)
    e[2] += int(kk)
    e[3] += int(kk) << int(mm)
out["by_m"] = {k: {"groups": v[0], "strings_in": v[1], "classes": v[2], "points": v[3]} for k, v in sorted(by_m.items())}
out["input_size_log2"] = dict(sorted(collections.Counter(int(np.log2(cc)) for cc in cnt).items()))
out["single_string_groups"] = int((cnt == 1).sum())
print(json.dumps(out), flush=True)
