"""Debug: fused / unfused engines vs the oracle, test ordering."""
import gc
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2506_13241_b200 as pp  # noqa: E402

geom = pp.heavy_hex_127()
init = O.site_word(62, 3)[None]
if "chain" in sys.argv:
    text = "\n".join(f"{i} {i + 1} {i % 2}" for i in range(63))
    e = pp.Engine(64, 0.0)
    e.set_initial(O.site_word(32, 3)[None], np.array([1.0]))
    e.run_circuit(pp.build_kicked_ising(pp.load_geometry(text), 0.3, "-0.5pi", 7))
    del e
    gc.collect()
if "prewarm" in sys.argv:
    e = pp.Engine(127, 0.0)
    e.set_initial(init, np.array([1.0]))
    e.run_circuit(pp.build_kicked_ising(geom, "0.25pi", "-0.5pi", 5))
    del e
    gc.collect()
circ = pp.build_kicked_ising(geom, "0.25pi", "-0.5pi", 4)
ora = O.OracleEngine(127, 0.0)
ora.set_initial(init, [1.0])
gates = [(np.asarray(g.generator.words), g.cos_theta, g.sin_theta) for g in circ.layers[0]]
orow = ora.run_layers(gates, 4)
ow, oc = ora.export()
a = pp.Engine(127, 0.0, fuse_clifford=True)
b = pp.Engine(127, 0.0, fuse_clifford=False)
for e in (a, b):
    e.set_initial(init, np.array([1.0]))
ra, rb = a.run_circuit(circ), b.run_circuit(circ)
for nm, e, rows in (("fused", a, ra), ("unfused", b, rb)):
    w, c = e.export()
    same = w.shape == ow.shape and (w == ow).all() and (c.view(np.uint64) == oc.view(np.uint64)).all()
    print(f"{nm} env={sys.argv[1:]} same={same}", [r["term_count"] for r in rows], [r["removed"] for r in rows],
          [o["term_count"] for o in orow])
    if not same and w.shape == ow.shape:
        bad = np.nonzero((w != ow).any(axis=1))[0]
        print("  differing rows", bad.size, bad[:5])
