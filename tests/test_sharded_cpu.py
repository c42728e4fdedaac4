"""The sharded (multi-rank) protocol on CPU: ownership by z-plane hash,
eviction/exchange/ingest after z-changing gates, global truncation threshold,
global sums.  Each rank's local engine is the oracle restatement
(tests/sharded_oracle.py); the result must equal one oracle engine run bit
for bit, for any rank count (the reference's worker-independence contract,
test_engine.cpp:211-258).  Ranks run as threads (ThreadComm) and, for the
real multi-process path, as world_size-2 gloo processes (TorchComm)."""
import json
import math
import os
import threading

import numpy as np
import pytest

from conftest import ROOT, assert_same_terms, gate_tuples

GOLD = os.path.join(ROOT, "tests", "golden")


def ref_geometry_text():
    lines = [l for l in open(os.path.join(GOLD, "heavy_hex_ref_order.txt")) if l.strip() and not l.startswith("#")]
    return "".join(lines)


def single_oracle(O, n, circ, init, eps, cadence):
    ora = O.OracleEngine(n, eps, 1 if cadence == "layer" else 0)
    ora.set_initial(np.stack([w for w, _ in init]), [c for _, c in init])
    L = circ.num_layers()
    for t in range(1, L + 1):
        for g in reversed(gate_tuples(circ.layers[L - t])):
            ora.apply_gate(*g)
        if cadence == "layer":
            ora.truncate_now()
    return ora


def run_sharded_threads(pp, n, circ, init, eps, cadence, world):
    from paper_2506_13241_b200.sharded import ShardedEngine, ThreadComm
    from sharded_oracle import OracleShard

    comms = ThreadComm.make(world)
    results, errors = [None] * world, []

    def rank_main(r):
        try:
            se = ShardedEngine(OracleShard(n, eps), n, comms[r], eps, cadence)
            se.set_initial(np.stack([w for w, _ in init]), [c for _, c in init])
            rows = se.run_circuit(circ)
            w, c = se.export()
            results[r] = (rows, w, c, se.exchanged_records)
        except Exception as exc:  # pragma: no cover - surfaced below
            errors.append(exc)
            comms[r].hub.barrier.abort()

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return results


CASES = [
    # (name, n, geometry, theta_x, theta_zz, init sites, eps, cadence, layers)
    ("hh_pi4_eps0", 127, "hh", "0.25pi", "-0.5pi", [62], 0.0, "gate", 4),
    ("hh_0.3_eps1e-4", 127, "hh", 0.3, "-0.5pi", [62], 1e-4, "gate", 4),
    ("hh_0.3_eps1e-3_layer", 127, "hh", 0.3, "-0.5pi", [62], 1e-3, "layer", 4),
    ("chain12_noncliff_zz", 12, "chain", 0.4, -math.pi / 2 + 0.2, list(range(12)), 1e-3, "gate", 3),
    ("chain64_0.3", 64, "chain", 0.3, "-0.5pi", [32], 0.0, "gate", 4),
]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_sharded_threads_match_single(pp, O, case, world):
    name, n, geom, thx, thzz, sites, eps, cadence, layers = case
    if geom == "hh":
        g = pp.load_geometry(ref_geometry_text())
    else:
        g = pp.load_geometry("\n".join(f"{i} {i + 1} {i % 2}" for i in range(n - 1)))
    circ = pp.build_kicked_ising(g, thx, thzz, layers)
    init = [(O.site_word(s, 3), 1.0 / len(sites)) for s in sites]
    ora = single_oracle(O, n, circ, init, eps, cadence)
    ow, oc = ora.export()
    res = run_sharded_threads(pp, n, circ, init, eps, cadence, world)
    for r in range(world):
        rows, w, c, _ = res[r]
        assert_same_terms(w, c, ow, oc, f"{name} world={world} rank={r}")
        assert rows[-1]["term_count"] == ora.term_count()
        assert abs(rows[-1]["observable"] - ora.expectation()) <= 1e-12 * max(1.0, abs(ora.expectation()))
    assert sum(res[r][3] for r in range(world)) > 0 or layers == 0  # strings did move between ranks


def test_shard_owner_is_a_pure_function_of_z(pp, O):
    rng = np.random.default_rng(9)
    words = rng.integers(0, 2**63, size=(500, 4), dtype=np.uint64)
    x, z = O.to_planes(words)
    # same z, different x -> same owner
    other = O.from_planes(x ^ np.uint64(0x5A5A), z)
    from paper_2506_13241_b200.sharded import SHARD_SEED
    a = pp._impl.shard_owner(words, 128, SHARD_SEED, 8)
    b = pp._impl.shard_owner(other, 128, SHARD_SEED, 8)
    assert (a == b).all()
    assert set(np.unique(a)) <= set(range(8)) and len(np.unique(a)) == 8


def _gloo_rank(rank, world, port, n, circ_spec, out_path):
    import torch.distributed as dist
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import paper_2506_13241_b200 as pp
    from paper_2506_13241_b200.sharded import ShardedEngine, TorchComm
    import oracle as O
    from sharded_oracle import OracleShard

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    thx, eps, layers = circ_spec
    g = pp.load_geometry(ref_geometry_text())
    circ = pp.build_kicked_ising(g, thx, "-0.5pi", layers)
    se = ShardedEngine(OracleShard(n, eps), n, TorchComm(), eps, "gate")
    se.set_initial(O.site_word(62, 3)[None], [1.0])
    rows = se.run_circuit(circ)
    w, c = se.export()
    if rank == 0:
        np.savez(out_path, w=w, c=c, tc=rows[-1]["term_count"], ob=rows[-1]["observable"])
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gloo_world2_matches_single(pp, O, tmp_path):
    import socket
    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "res.npz")
    spec = (0.3, 1e-4, 4)
    mp.spawn(_gloo_rank, args=(2, port, 127, spec, out), nprocs=2, join=True)
    res = np.load(out)
    g = pp.load_geometry(ref_geometry_text())
    circ = pp.build_kicked_ising(g, spec[0], "-0.5pi", spec[2])
    ora = single_oracle(O, 127, circ, [(O.site_word(62, 3), 1.0)], spec[1], "gate")
    ow, oc = ora.export()
    assert_same_terms(res["w"], res["c"], ow, oc, "gloo world=2")
    assert int(res["tc"]) == ora.term_count()


def _run_threads(world, fn):
    from paper_2506_13241_b200.sharded import ThreadComm
    comms = ThreadComm.make(world)
    results, errors = [None] * world, []

    def main(r):
        try:
            results[r] = fn(comms[r])
        except Exception as exc:  # pragma: no cover
            errors.append(exc)
            comms[r].hub.barrier.abort()

    th = [threading.Thread(target=main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    return results


def test_sharded_histogram_and_checkpoint_resume(pp, O, tmp_path):
    """Global histogram = the single engine's (counts summed over ranks);
    a checkpoint written by 3 ranks resumes on 2 ranks and finishes with the
    single-engine result bit for bit."""
    from paper_2506_13241_b200.sharded import ShardedEngine
    from sharded_oracle import OracleShard

    n, eps, L, k = 127, 1e-4, 4, 2
    g = pp.load_geometry(ref_geometry_text())
    circ = pp.build_kicked_ising(g, 0.3, "-0.5pi", L)
    init = [(O.site_word(62, 3), 1.0)]
    ora = single_oracle(O, n, circ, init, eps, "gate")
    ow, oc = ora.export()
    pos, neg = ora.density_histogram(16, eps)
    want_tsv = pp.histogram_from_counts(16, eps, pos.tolist(), neg.tolist())["tsv"]
    out = str(tmp_path / "run")

    def first(comm):
        se = ShardedEngine(OracleShard(n, eps), n, comm, eps, "gate")
        se.set_initial(O.site_word(62, 3)[None], [1.0])
        se.run_circuit(circ, out_dir=out, histogram_bins=16, checkpoint_every=k)
        return se.density_histogram(16)["tsv"]

    tsvs = _run_threads(3, first)
    assert all(t == want_tsv for t in tsvs)
    assert open(os.path.join(out, f"histogram_t{L}.tsv")).read() == want_tsv
    man = json.load(open(os.path.join(out, f"checkpoint_t{k}", "manifest.json")))
    assert len(man["files"]) == 3 and man["layer"] == k

    def second(comm):
        se = ShardedEngine(OracleShard(n, eps), n, comm, eps, "gate")
        assert se.load_checkpoint(os.path.join(out, f"checkpoint_t{k}")) == k
        rows = se.run_circuit(circ, start_layer=k)
        return rows, se.export()

    for rows, (w, c) in _run_threads(2, second):
        assert [r["t"] for r in rows] == list(range(k + 1, L + 1))
        assert_same_terms(w, c, ow, oc, "sharded resume 3 -> 2 ranks")
