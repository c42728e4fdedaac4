"""The native sharded engine (C-ABI pp_sharded_*, include/pauliprop_gpu.h):
SPMD ranks with bucket-balanced z-hash ownership, device all-to-all
exchange after string-moving steps and per-run reduced speculative Rx runs
for eps0 > 0.  On the one GPU this environment reaches, ranks run as threads
sharing the device through the in-process hub transport (host barriers and
device-to-device copies -- no kernel waits on another rank); the NCCL
transport is exercised with one rank.  Every case must reproduce the
single-engine run bit for bit: the union of the ranks' strings and
coefficient bits, the term count, the global max and the summed counters."""
import math
import threading

import numpy as np
import pytest

from conftest import assert_same_terms

pytestmark = pytest.mark.gpu


def _single(pp, O, n, eps, circ, init):
    eng = pp.Engine(n, eps)
    eng.set_initial(np.stack([w for w, _ in init]), np.array([c for _, c in init]))
    rows = eng.run_circuit(circ)
    return eng.export(), rows


def _sharded(pp, n, eps, circ, init, world):
    hub = pp.ShardHub(world)
    out = [None] * world
    err = [None] * world
    words = np.stack([w for w, _ in init])
    coeffs = np.array([c for _, c in init])

    def rank_main(r):
        try:
            e = pp.NativeShardedEngine(n, eps, "gate", world=world, rank=r, hub=hub)
            e.set_initial(words, coeffs)
            rows = e.run_circuit(circ)
            out[r] = (e.local_export(), rows, e.stats())
        except Exception as x:  # noqa: BLE001
            err[r] = x

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for x in err:
        if x is not None:
            raise x
    w = np.concatenate([o[0][0] for o in out])
    c = np.concatenate([o[0][1] for o in out])
    order = np.lexsort((w[:, 0], w[:, 1], w[:, 2], w[:, 3]))
    return (w[order], c[order]), [o[1] for o in out], [o[2] for o in out]


CASES = {
    "config1_eps0": (127, 0.0, "0.25pi", "-0.5pi", 4, "z62"),
    "hh_pi4_eps1e-4": (127, 1e-4, "0.25pi", "-0.5pi", 6, "z62"),
    "config4_shape": (127, 1e-4, 0.4, -math.pi / 2 + 0.2, 3, "sum"),
    "chain64_eps0": (64, 0.0, 0.3, "-0.5pi", 6, "z32"),
}


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", sorted(CASES))
def test_hub_ranks_match_single_engine(pp, O, name, world):
    n, eps, tx, tz, layers, obs = CASES[name]
    geom = pp.heavy_hex_127() if n == 127 else pp.load_geometry("\n".join(f"{i} {i + 1} {i % 2}" for i in range(63)))
    circ = pp.build_kicked_ising(geom, tx, tz, layers)
    if obs == "sum":
        init = [(O.site_word(q, 3), 1.0 / 127) for q in range(127)]
    else:
        init = [(O.site_word(int(obs[1:]), 3), 1.0)]
    (sw, sc), srows = _single(pp, O, n, eps, circ, init)
    (hw, hc), hrows, stats = _sharded(pp, n, eps, circ, init, world)
    assert_same_terms(hw, hc, sw, sc, f"{name} world {world}")
    for r in range(world):
        for a, b in zip(hrows[r], srows):
            assert a["term_count"] == b["term_count"]
            assert a["global_max"] == b["global_max"]
            assert a["records_sent"] == b["records_sent"] and a["removed"] == b["removed"]
            assert abs(a["observable"] - b["observable"]) <= 1e-12 * max(1.0, abs(b["observable"]))
    assert all(s["exchanges"] > 0 for s in stats)


def test_nccl_transport_one_rank(pp, O):
    """The NCCL transport end to end (unique id, communicator, all-reduce,
    grouped send/recv) with one rank: identical to the single engine."""
    geom = pp.heavy_hex_127()
    circ = pp.build_kicked_ising(geom, "0.25pi", "-0.5pi", 5)
    init = [(O.site_word(62, 3), 1.0)]
    (sw, sc), srows = _single(pp, O, 127, 1e-5, circ, init)
    e = pp.NativeShardedEngine(127, 1e-5, "gate", world=1, rank=0, nccl_id=pp.nccl_unique_id())
    e.set_initial(np.stack([w for w, _ in init]), np.array([1.0]))
    rows = e.run_circuit(circ)
    w, c = e.local_export()
    assert_same_terms(w, c, sw, sc, "nccl world 1")
    assert [r["term_count"] for r in rows] == [r["term_count"] for r in srows]
