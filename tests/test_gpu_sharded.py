"""Sharded GPU engines (one per emulated rank, threads on one B200) against a
single engine: same string set and coefficients bit for bit.  The exchange
runs host-staged or device-resident (engine device buffers exchanged by
device copies, the data flow of the NCCL all-to-all); either way no kernel
waits on another rank."""
import math
import threading

import numpy as np
import pytest

from conftest import assert_same_terms

pytestmark = pytest.mark.gpu


def run_sharded(pp, n, circ, init_words, init_coeffs, eps, cadence, world, device=False):
    from paper_2506_13241_b200.sharded import GpuShard, ShardedEngine, ThreadComm

    comms = ThreadComm.make(world, device=device)
    results, errors = [None] * world, []

    def rank_main(r):
        try:
            se = ShardedEngine(GpuShard(n, eps, cadence), n, comms[r], eps, cadence)
            se.set_initial(init_words, init_coeffs)
            rows = se.run_circuit(circ)
            results[r] = (rows, *se.export(), se.exchanged_records)
        except Exception as exc:  # pragma: no cover
            errors.append(exc)
            comms[r].hub.barrier.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    return results


@pytest.mark.parametrize("device", [False, True], ids=["host_staged", "device_exchange"])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", [
    ("hh_pi4_eps0", 127, "0.25pi", "-0.5pi", 0.0, "gate", 5),
    ("hh_0.3_eps1e-4", 127, 0.3, "-0.5pi", 1e-4, "gate", 5),
    ("hh_0.3_eps1e-3_layer", 127, 0.3, "-0.5pi", 1e-3, "layer", 4),
    ("hh_noncliff_zz", 127, 0.4, -math.pi / 2 + 0.2, 1e-4, "gate", 3),
], ids=lambda c: c[0] if isinstance(c, tuple) else str(c))
def test_sharded_gpu_matches_single(pp, O, case, world, device):
    name, n, thx, thzz, eps, cadence, layers = case
    geom = pp.heavy_hex_127()
    circ = pp.build_kicked_ising(geom, thx, thzz, layers)
    if name == "hh_noncliff_zz":
        words = np.stack([O.site_word(q, 3) for q in range(127)])
        coeffs = np.full(127, 1.0 / 127)
    else:
        words = O.site_word(62, 3)[None]
        coeffs = np.array([1.0])
    single = pp.Engine(n, eps, cadence)
    single.set_initial(words, coeffs)
    srows = single.run_circuit(circ)
    sw, sc = single.export()
    res = run_sharded(pp, n, circ, words, coeffs, eps, cadence, world, device)
    for r in range(world):
        rows, w, c, _ = res[r]
        assert_same_terms(w, c, sw, sc, f"{name} world={world} rank={r}")
        for a, b in zip(rows, srows):
            assert a["term_count"] == b["term_count"]
            assert abs(a["observable"] - b["observable"]) <= 1e-12 * max(1.0, abs(b["observable"]))
    assert sum(x[3] for x in res) > 0


def test_sharded_gpu_histogram_and_resume(pp, O, tmp_path):
    """Device histograms summed over 2 ranks equal the single engine's TSV;
    a 2-rank checkpoint resumes on 3 ranks to the single engine's result."""
    from paper_2506_13241_b200.sharded import GpuShard, ShardedEngine, ThreadComm

    n, eps, L, k = 127, 1e-4, 5, 3
    circ = pp.build_kicked_ising(pp.heavy_hex_127(), 0.3, "-0.5pi", L)
    z62 = O.site_word(62, 3)[None]
    single = pp.Engine(n, eps, "gate")
    single.set_initial(z62, [1.0])
    single.run_circuit(circ)
    sw, sc = single.export()
    want = single.density_histogram(32)["tsv"]
    out = str(tmp_path / "run")

    def run(world, fn):
        comms = ThreadComm.make(world)
        res, errs = [None] * world, []

        def main(r):
            try:
                res[r] = fn(comms[r])
            except Exception as exc:  # pragma: no cover
                errs.append(exc)
                comms[r].hub.barrier.abort()

        th = [threading.Thread(target=main, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        return res

    def first(comm):
        se = ShardedEngine(GpuShard(n, eps, "gate"), n, comm, eps, "gate")
        se.set_initial(z62, [1.0])
        se.run_circuit(circ, out_dir=out, histogram_bins=32, checkpoint_every=k, binary_checkpoint=True)
        return se.density_histogram(32)["tsv"]

    assert all(t == want for t in run(2, first))

    def second(comm):
        se = ShardedEngine(GpuShard(n, eps, "gate"), n, comm, eps, "gate")
        assert se.load_checkpoint(f"{out}/checkpoint_t{k}") == k
        se.run_circuit(circ, start_layer=k)
        return se.export()

    for w, c in run(3, second):
        assert_same_terms(w, c, sw, sc, "gpu sharded resume 2 -> 3 ranks")
