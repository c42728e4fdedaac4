#!/usr/bin/env python
"""Benchmark of the Heisenberg-picture Pauli-propagation hot path on B200.

Metric (BASELINE.json): Pauli-string terms processed per second per gate
layer = string-gates/s, where one string-gate is one live string entering
one gate.  Sum over gates of |O_in| / time.

Workload (default): BASELINE.json config 0 in full -- the 64-qubit open
kicked-Ising chain, theta_h = 0.3, theta_J = -pi/2, O0 = Z32, eps0 = 0, all
10 Trotter steps (final |O| = 987,369,656 strings, ~24 GB of live state):
the largest BASELINE configuration that runs on one B200 at eps0 = 0.  One
bench step = one full propagation from O0 (1,270 gates), readout after every
layer, exactly what the reference's run_circuit does.  Other workloads:
``--workload config1`` (BASELINE configs[1]), ``config0_t9``,
``config2_pi4_eps1e-4_t8``.

  value -- device-timed (CUDA events on the engine's stream), state created
           on the device, string-gates/s
  e2e   -- the public API call a user makes (simulate(...)), host circuit
           in, ledger rows out, wall-clocked around the call
  cpu_baseline -- the reference engine compiled from its own sources
           (oracle/_ref), on this box's host cores, on the largest prefix of
           the workload it runs in seconds (config 0 to t = 9, 81.7 M strings)

``--impl reference`` times the reference CPU engine on the same workload.
``--gpus N`` relaunches itself under torch.distributed.run; with N > 1 ranks
the operator is sharded by the native engine (C-ABI pp_sharded_*, NCCL
inside): Rx runs are rank-local, strings move with one all-to-all after each
Clifford run, scalars are all-reduced -- total work fixed, strong scaling
(DESIGN.md section 6).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# name: (geometry, n, theta_x, theta_zz, observable site, eps0, layers)
WORKLOADS = {
    "config1": ("heavy_hex", 127, "0.25pi", "-0.5pi", 62, 0.0, 5),
    "config0_t8": ("chain64", 64, 0.3, "-0.5pi", 32, 0.0, 8),
    "config0_t9": ("chain64", 64, 0.3, "-0.5pi", 32, 0.0, 9),
    "config0_t10": ("chain64", 64, 0.3, "-0.5pi", 32, 0.0, 10),
    "config2_pi4_eps1e-4_t8": ("heavy_hex", 127, "0.25pi", "-0.5pi", 62, 1e-4, 8),
}
# Exact sum over gates of |O_in| (string-gates per step) and the final |O|,
# counted once gate by gate (``--count`` recounts; tests pin the small ones
# against the reference engine's own count).
COUNTS = {
    "config1": (106882582, 2146372),
    "config0_t8": (283416094, 6952660),
    "config0_t9": (3242286702, 81662152),
    "config0_t10": (38261630218, 987369656),
    "config2_pi4_eps1e-4_t8": (4518354553, 11856422),
}
# The reference CPU engine cannot hold config 0 at t = 10 (~1e9 strings) in a
# few minutes: its arm and cpu_baseline time the largest prefix that runs in
# seconds per step on the box's host cores.
CPU_SAMPLE = {"config0_t10": "config0_t9"}
DEFAULT_WORKLOAD = "config0_t10"


def chain_text(n):
    return "\n".join(f"{i} {i + 1} {i % 2}" for i in range(n - 1))


def build_circuit(pp, wl):
    geom_kind, n, thx, thzz, site, eps, layers = wl
    geom = pp.heavy_hex_127() if geom_kind == "heavy_hex" else pp.load_geometry(chain_text(64))
    return pp.build_kicked_ising(geom, thx, thzz, layers)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region: NVML
    polled every ~1 ms from a thread (a timed region of a few ms still gets
    samples), nvidia-smi -lms as the fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, device):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, set of reasons)
        self.stop = threading.Event()
        self.t = None
        self.nvml = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        self.nvml = pynvml
        try:
            import torch
            p = torch.cuda.get_device_properties(self.device)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = int(vis.split(",")[self.device]) if vis and vis.split(",")[0].isdigit() else self.device
            return pynvml.nvmlDeviceGetHandleByIndex(idx)

    def _poll(self, h):
        nv = self.nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, mx, {nm for nm, a in self.REASONS if r & getattr(nv, a)}))
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        try:
            h = self._handle()
            self.t = threading.Thread(target=self._poll, args=(h,), daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=5)

    def summary(self):
        sm = sorted(s[0] for s in self.samples)
        reasons = set()
        for s in self.samples:
            reasons |= s[2]
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": max((s[1] for s in self.samples), default=None),
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvml, ~1 ms polling"}


def string_gates(pp, circ, wl):
    """Exact sum over gates of |O_in| for the workload (one counted run,
    outside every timed region)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    n, site, eps = wl[1], wl[4], wl[5]
    eng = pp.Engine(n, eps)
    w = np.zeros((1, 4), np.uint64)
    w[0, site // 32] = np.uint64(3) << np.uint64(2 * (site % 32))
    eng.set_initial(w, np.array([1.0]))
    total = 0
    L = circ.num_layers()
    for t in range(1, L + 1):
        layer = circ.layers[L - t]
        for g in reversed(layer):
            total += eng.term_count()
            eng.apply_gate(g)
    return total, eng.term_count()


def cpu_reference_time(wl, steps, warmup, threads):
    """Reference CPU engine (oracle/_ref, compiled from the reference's own
    sources) on the same workload; returns (seconds per step list, string_gates)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import oracle as O
    geom_kind, n, thx, thzz, site, eps, layers = wl
    if geom_kind == "heavy_hex":
        edges, cols = O.ref_heavy_hex()
        text = "\n".join(f"{a} {b} {c}" for (a, b), c in zip(edges, cols))
    else:
        text = chain_text(64)
    words, is_zz = O.ref_kicked_layer(text)

    def ang(v):
        if isinstance(v, str):
            return float(v[:-2]), 1
        return float(v), 0
    ax, az = ang(thx), ang(thzz)
    gates = [(words[i], az[0] if is_zz[i] else ax[0], az[1] if is_zz[i] else ax[1]) for i in range(len(is_zz))]
    init = np.zeros((1, 4), np.uint64)
    init[0, site // 32] = np.uint64(3) << np.uint64(2 * (site % 32))
    times, sg = [], 0.0
    for i in range(warmup + steps):
        r = O.RefEngine(n, eps, workers=threads, threads=threads)
        r.set_initial(init, [1.0])
        sec, sg = r.time_circuit(gates, layers)
        if i >= warmup:
            times.append(sec)
        del r
    return times, sg


def config_dict(args, wl, world):
    """The `config` object both arms print (same keys, same values)."""
    sg, final_terms = COUNTS[args.workload]
    return {"workload": args.workload, "epsilon0": wl[5], "layers": wl[6], "string_gates_per_step": sg,
            "final_terms": final_terms, "observable": f"Z{wl[4]}", "n_qubits": wl[1],
            "l2": "flushed (512 MB write) before every timed step and every e2e call",
            "parallelism": "single GPU" if world == 1 else f"z-hash shards x{world}"}


def cpu_sample_note(name, threads, runs):
    return (f"{name}: full propagation per step through the reference engine compiled from its sources "
            f"(oracle/_ref, -O3), {threads} workers = threads, median of {runs}")


def run_reference_arm(args, wl, rank, world):
    """The reference's own CPU engine on the host cores, rank 0 only.  For a
    workload the reference cannot run in seconds (config0_t10) each step is
    the largest prefix that does (CPU_SAMPLE), stated in cpu_baseline.sample."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample = CPU_SAMPLE.get(args.workload, args.workload)
    times, sg = cpu_reference_time(WORKLOADS[sample], args.steps, args.warmup, threads)
    per = sorted(times)[len(times) // 2]
    value = sg / per
    line = {
        "metric": "string_gates_per_s", "value": value, "unit": "string-gates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic circuit)",
        "impl": "reference",
        "config": config_dict(args, wl, world),
        "cpu_baseline": {"value": value, "unit": "string-gates/s", "cores": threads, "kind": "reference",
                         "sample": cpu_sample_note(sample, threads, len(times)),
                         "sample_string_gates_per_step": sg},
        "e2e": {"value": value, "unit": "string-gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_sharded(args, pp, circ, wl, sg, final_terms, init, rank, world, local):
    """N > 1: the native sharded engine (C-ABI pp_sharded_*: NCCL inside,
    bucket-balanced z-hash ownership, one all-to-all per string-moving step,
    per-run reduced speculation for eps0 > 0).  torch.distributed only
    bootstraps it (broadcast of the NCCL id) and takes the max over ranks of
    the timings.  Total work fixed -> strong scaling."""
    import numpy as np
    import torch
    import torch.distributed as dist

    n, site, eps = wl[1], wl[4], wl[5]
    gloo = dist.group.WORLD
    idt = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        idt = torch.tensor(list(pp.nccl_unique_id()), dtype=torch.uint8)
    dist.broadcast(idt, 0, group=gloo)
    eng = pp.NativeShardedEngine(n, eps, "gate", world=world, rank=rank, nccl_id=bytes(idt.tolist()), device=local)
    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=local)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    def one_step():
        eng.set_initial(init, np.array([1.0]))
        return eng.run_circuit(circ)

    for _ in range(args.warmup):
        one_step()
    eng.kernel_stats()
    st0 = eng.stats()
    ms, walls, rows = [], [], None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier(group=gloo)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            t0 = time.perf_counter()
            rows = one_step()
            e1.record(stream)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
            ms.append(e0.elapsed_time(e1))
    ks = eng.kernel_stats()
    st1 = eng.stats()
    assert rows[-1]["term_count"] == final_terms, (rows[-1]["term_count"], final_terms)
    red = torch.tensor([sum(ms), sum(walls), ks["branch_ms"], ks["branch_bytes"],
                        float(st1["records_moved"] - st0["records_moved"]),
                        (st1["exchange_ns"] - st0["exchange_ns"]) * 1e-6], dtype=torch.float64)
    mx = red.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=gloo)
    tot = red.clone()
    dist.all_reduce(tot, op=dist.ReduceOp.SUM, group=gloo)
    ms_per_step = float(mx[0]) / args.steps
    wall_per_step = float(mx[1]) / args.steps
    if rank == 0:
        peak, peak_kind = load_peaks()
        achieved = float(tot[3]) / (float(mx[2]) / 1e3) / 1e9 / world if mx[2] > 0 else 0.0  # per GPU
        moved_bytes = float(mx[4]) * eng.record_bytes() / args.steps
        ex_ms = float(mx[5]) / args.steps
        line = {
            "metric": "string_gates_per_s", "value": sg / (ms_per_step / 1e3), "unit": "string-gates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (deterministic kicked-Ising circuit, BASELINE config; no dataset)",
            "config": config_dict(args, wl, world),
            "e2e": {"value": sg / wall_per_step, "unit": "string-gates/s", "h2d_bytes_per_step": 40,
                    "d2h_bytes_per_step": 8 * 4 * circ.num_layers(), "api": "NativeShardedEngine.run_circuit",
                    "bytes": "the initial term in, four ledger scalars per layer out"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None, "traffic": None, "peak_kind": peak_kind,
                         "kernel": "k_dense_sublayer + k_branch_sublayer (per GPU, summed bytes / max device time)",
                         "exchange": {"bound": "nvlink", "bytes_per_step_max_rank": moved_bytes,
                                      "ms_per_step_max_rank": ex_ms,
                                      "achieved_GBps": moved_bytes / (ex_ms / 1e3) / 1e9 if ex_ms > 0 else None,
                                      "peak_GBps": 900.0,
                                      "note": "exchange time includes the rebalance all-reduce and the ingest"}},
            "cpu_baseline": None,
            "clocks": clk.summary(),
            "gpu_launches": int(ks["launches"]),
        }
        print(json.dumps(line), flush=True)
    dist.barrier(group=gloo)
    dist.destroy_process_group()


def spawn_ranks(args):
    """``--gpus N`` outside torchrun: relaunch this script under
    torch.distributed.run with N ranks (one per GPU) on 127.0.0.1."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--count", action="store_true", help="recount string-gates gate by gate (slow)")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, wl, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:  # bootstrap and timing reductions only; the data plane is NCCL inside the engine
        dist.init_process_group("gloo")

    import paper_2506_13241_b200 as pp

    circ = build_circuit(pp, wl)
    n, site, eps = wl[1], wl[4], wl[5]
    if args.count:
        COUNTS[args.workload] = string_gates(pp, circ, wl)
    sg, final_terms = COUNTS[args.workload]
    init = np.zeros((1, 4), np.uint64)
    init[0, site // 32] = np.uint64(3) << np.uint64(2 * (site % 32))
    if world > 1:
        run_sharded(args, pp, circ, wl, sg, final_terms, init, rank, world, local)
        return

    # ---------------- device-resident value: CUDA events on the engine stream
    eng = pp.Engine(n, eps, device=local)
    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=local)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")  # > 126 MB L2

    def one_step():
        eng.set_initial(init, np.array([1.0]))
        return eng.run_circuit(circ)

    for _ in range(args.warmup):
        one_step()
    eng.kernel_stats()
    ms = []
    rows = None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rows = one_step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
    ks = eng.kernel_stats()
    assert rows[-1]["term_count"] == final_terms, (rows[-1]["term_count"], final_terms)
    ms_per_step = sum(ms) / args.steps
    value = sg / (ms_per_step / 1e3)
    # roofline pass (untimed): no graphs, CUDA events around every branch launch
    del eng, stream  # its device buffers return to the engine's pool for reuse
    import gc
    gc.collect()
    peng = pp.Engine(n, eps, device=local, profile=True)
    peng.set_initial(init, np.array([1.0]))
    peng.kernel_stats()
    peng.run_circuit(circ)
    pks = peng.kernel_stats()
    del peng
    gc.collect()

    # ---------------- e2e through the public API (simulate): host circuit in,
    # ledger rows out, L2 flushed before every call, bytes counted by the engine
    e2e_times, h2d, d2h = [], [], []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        b0 = pp.transfer_totals()
        t0 = time.perf_counter()
        out = pp.simulate(circ, observable=f"Z{site}", epsilon0=eps)
        t1 = time.perf_counter()
        b1 = pp.transfer_totals()
        if i >= args.warmup:
            e2e_times.append(t1 - t0)
            h2d.append(b1[0] - b0[0])
            d2h.append(b1[1] - b0[1])
    assert out[-1]["term_count"] == final_terms
    e2e_sorted = sorted(e2e_times)
    e2e_s = e2e_sorted[len(e2e_sorted) // 2]  # median: one engine per call, robust to host hiccups
    e2e_value = sg / e2e_s

    peak, peak_kind = load_peaks()
    achieved = pks["branch_bytes"] / (pks["branch_ms"] / 1e3) / 1e9 if pks["branch_ms"] > 0 else 0.0
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "branch_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                tr = json.load(f).get(args.workload)
            if tr:  # ncu DRAM bytes per launch of the same kernel (tools/traffic.py)
                traffic = tr["dram_bytes_per_launch"]
                traffic_src = tr
        except Exception:
            traffic = None

    cpu = None
    if not args.no_cpu_baseline:
        sample = CPU_SAMPLE.get(args.workload, args.workload)
        try:
            threads = os.cpu_count() or 1
            times, csg = cpu_reference_time(WORKLOADS[sample], 1, 1, threads)
            cpu = {"value": csg / times[0], "unit": "string-gates/s", "cores": threads, "kind": "reference",
                   "sample": cpu_sample_note(sample, threads, 1) + " after 1 warm-up run",
                   "sample_string_gates_per_step": csg}
        except Exception as exc:  # the reference build travels as oracle/_ref
            cpu = {"value": None, "unit": "string-gates/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    R = 16 * ((n + 63) // 64) + 8  # SURVEY 8d streaming record: x, z planes + coefficient
    line = {
        "metric": "string_gates_per_s", "value": value, "unit": "string-gates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic kicked-Ising circuit, BASELINE config; no dataset)",
        "config": config_dict(args, wl, world),
        "e2e": {"value": e2e_value, "unit": "string-gates/s",
                "h2d_bytes_per_step": int(sorted(h2d)[len(h2d) // 2]),
                "d2h_bytes_per_step": int(sorted(d2h)[len(d2h) // 2]),
                "bytes": "counted by the engine (pp_transfer_totals): every copy + parameter blocks carrying "
                         "host data", "ms_per_step": e2e_s * 1e3, "api": "simulate()",
                "stat": "median over steps", "ms_min": e2e_sorted[0] * 1e3,
                "ms_mean": sum(e2e_times) / len(e2e_times) * 1e3},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per launch (ncu)",
                     "algorithmic_bytes_per_launch": (pks["branch_bytes"] / pks["branch_launches"]
                                                      if pks["branch_launches"] else None),
                     "traffic_detail": traffic_src,
                     "kernel": "k_dense_sublayer (+ k_branch_sublayer for the groups it leaves; k_branch_x on per-gate launches)", "peak_kind": peak_kind,
                     "bytes_model": "(strings read + strings written) x (8W+8) B per launch; the dense "
                                    "sublayer reads each input string once and writes each output "
                                    "string once per Rx run",
                     "branch_ms_per_step": pks["branch_ms"],
                     "branch_share_of_step": pks["branch_ms"] / ms_per_step,
                     "branch_bytes_per_step": pks["branch_bytes"],
                     "branch_launches_per_step": pks["branch_launches"],
                     "how": "separate untimed pass, CUDA events around each Rx-run launch (pair) on the engine stream",
                     "streaming_model": {
                         "bytes_per_string_gate": 2 * R,
                         "equivalent_GBps": value * 2 * R / 1e9,
                         "note": "SURVEY 8d per-gate streaming bytes; the fused runs touch each string once "
                                 "per run, so this equivalent exceeds HBM peak"}},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": int(ks["launches"]),
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
