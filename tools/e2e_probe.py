"""simulate() wall time per call for a bench workload (e2e variance probe).
  python tools/e2e_probe.py [workload] [calls]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_13241_b200 as pp  # noqa: E402

wl_name = sys.argv[1] if len(sys.argv) > 1 else "config0_t10"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 12
wl = bench.WORKLOADS[wl_name]
circ = bench.build_circuit(pp, wl)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")
for i in range(calls):
    flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = pp.simulate(circ, observable=f"Z{wl[4]}", epsilon0=wl[5])
    t1 = time.perf_counter()
    print(f"call {i}: {1e3 * (t1 - t0):.2f} ms  |O|={out[-1]['term_count']}", flush=True)
