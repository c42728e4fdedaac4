import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, bench
import paper_2506_13241_b200 as pp
wl = ("heavy_hex", 127, "0.25pi", "-0.5pi", 62, 1e-4, int(sys.argv[1]) if len(sys.argv) > 1 else 4)
circ = bench.build_circuit(pp, wl)
init = np.zeros((1, 4), np.uint64); init[0, 1] = np.uint64(3) << np.uint64(2 * (62 % 32))
e = pp.Engine(127, 1e-4); e.set_initial(init, np.array([1.0])); rows = e.run_circuit(circ)
print([r["term_count"] for r in rows])
