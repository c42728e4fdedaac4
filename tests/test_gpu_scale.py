"""Parity at the sizes the bench and DESIGN claim, through the public API
(pp.heavy_hex_127 / load_geometry -> build_kicked_ising -> Engine.run_circuit)
against fixtures the REFERENCE engine produced (tests/golden/scale.json,
tests/golden/ledgers.json; generators committed next to them):

* every ledger key but wall time, per layer, bit-exact for the integers and
  the global max, <O> to 1e-12 relative (BASELINE tolerance);
* SHA-256 of the whole sorted operator (words + coefficient bits) at chosen
  layers: config 0 to t = 9 (81,662,152 strings), heavy-hex pi/4 at
  eps0 = 1e-4 for all 20 steps, the config-4 shape to t = 8;
* config 0 at t = 10 (987,369,656 strings; the reference cannot hold it in
  this box's budget): sum c^2 = 1 (unitary, eps0 = 0), the term count, and
  sampled coefficients against a meet-in-the-middle evaluation with the
  oracle: c_P(O(10)) = sum_Q a_Q(5) b_Q with a = O(5) (Heisenberg) and
  b = U^5 P U^-5 (forward) for low-weight P, both small.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden")


def chain_geometry(pp, n=64):
    return pp.load_geometry("\n".join(f"{i} {i + 1} {i % 2}" for i in range(n - 1)))


def _angles(case):
    """(theta_x, theta_zz) as build_kicked_ising takes them; ledgers.json and
    scale.json spell the keys differently."""
    tx, txp = case.get("theta_x", case.get("thx")), case.get("theta_x_pi", case.get("thx_pi"))
    tz, tzp = case.get("theta_zz", case.get("thzz")), case.get("theta_zz_pi", case.get("thzz_pi"))
    return (f"{tx!r}pi" if txp else tx), (f"{tz!r}pi" if tzp else tz)


def _geometry(pp, case):
    return pp.heavy_hex_127() if case["geometry"] == "heavy_hex_ref" else chain_geometry(pp, case["n"])


def circuit_of(pp, case, layers=None):
    tx, tz = _angles(case)
    return pp.build_kicked_ising(_geometry(pp, case), tx, tz, layers or case["layers"])


def _eps(case):
    return case.get("epsilon0", case.get("eps"))


def init_of(O, case):
    w = np.stack([O.site_word(s, 3) for s, _ in case["init"]])
    return w, np.array([c for _, c in case["init"]])


def digest(words, coeffs):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(words, np.uint64).tobytes())
    h.update(np.ascontiguousarray(coeffs, np.float64).tobytes())
    return h.hexdigest()


def check_row(got, want, ctx):
    assert got["term_count"] == want["term_count"], ctx
    assert np.float64(got["global_max"]).view(np.uint64) == want["global_max_bits"], ctx
    assert got["removed"] == want["removed"], ctx
    assert got["records_sent"] == want["records_sent"], ctx
    assert got["batches_sent"] == want["batches_sent"], ctx
    assert abs(got["observable"] - want["observable"]) <= 1e-12 * max(1.0, abs(want["observable"])), ctx


def run_case(pp, O, case, cadence="gate"):
    """Layer by layer through Engine.run_circuit; yields (t, row, engine)."""
    eng = pp.Engine(case["n"], _eps(case), cadence)
    eng.set_initial(*init_of(O, case))
    one = circuit_of(pp, case, layers=1)
    for t in range(1, case["layers"] + 1):
        row = eng.run_circuit(one)[0]
        yield t, row, eng


@pytest.fixture(scope="module")
def scale():
    with open(os.path.join(GOLD, "scale.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def ledgers():
    with open(os.path.join(GOLD, "ledgers.json")) as f:
        return json.load(f)


def test_ledgers_through_public_api(pp, O, ledgers):
    """All 8 ledger keys (wall time aside) of every reference ledger case,
    run through pp.simulate with the package's own heavy_hex_127()."""
    for case in ledgers["cases"]:
        circ = circuit_of(pp, case)
        if len(case["init"]) == 1:
            rows = pp.simulate(circ, observable=f"Z{case['init'][0][0]}", epsilon0=_eps(case),
                               cadence="layer" if case["cadence"] else "gate")
        else:
            eng = pp.Engine(case["n"], _eps(case), "layer" if case["cadence"] else "gate")
            eng.set_initial(*init_of(O, case))
            rows = eng.run_circuit(circ)
        assert len(rows) == len(case["rows"])
        for got, want in zip(rows, case["rows"]):
            check_row(got, want, (case["name"], want["t"]))


@pytest.mark.parametrize("name", ["config4_eps1e-4_t8", "hh_pi4_eps1e-4_t20", "chain64_t9"])
def test_scale_case_bitexact(pp, O, scale, name):
    case = scale[name]
    for t, row, eng in run_case(pp, O, case):
        check_row(row, case["rows"][t - 1], (name, t))
        if str(t) in case["digests"]:
            w, c = eng.export()
            assert digest(w, c) == case["digests"][str(t)], (name, t, "operator digest")
            del w, c
    if name == "hh_pi4_eps1e-4_t20":
        # <Z62>(20) at theta_h = pi/4, eps0 = 1e-4
        assert abs(row["observable"] - 0.16417233944212911) <= 1e-12


def test_config0_t10_properties(pp, O):
    """BASELINE config 0 in full (987,369,656 strings at t = 10)."""
    geom = chain_geometry(pp)
    circ = pp.build_kicked_ising(geom, 0.3, "-0.5pi", 10)
    eng = pp.Engine(64, 0.0)
    eng.set_initial(O.site_word(32, 3)[None], np.array([1.0]))
    rows = eng.run_circuit(circ)
    assert rows[-1]["term_count"] == 987369656
    assert rows[8]["term_count"] == 81662152
    assert abs(eng.norm2() - 1.0) <= 1e-12  # unitary evolution, nothing truncated
    # meet in the middle: a = O(5) (Heisenberg, 5 steps), b_P = U^5 P U^-5
    layer = [(np.asarray(g.generator.words, np.uint64), g.cos_theta, g.sin_theta) for g in circ.layers[0]]
    A = O.OracleEngine(64, 0.0)
    A.set_initial(O.site_word(32, 3)[None], [1.0])
    A.run_layers(layer, 5)
    aw, ac = A.export()
    amap = {tuple(int(v) for v in k): float(x) for k, x in zip(aw, ac)}
    # candidates: the strings of O(3) (weight <= 5) -- small forward cones,
    # and live in O(10) unless a coefficient cancels exactly
    B3 = O.OracleEngine(64, 0.0)
    B3.set_initial(O.site_word(32, 3)[None], [1.0])
    B3.run_layers(layer, 3)
    cw, _ = B3.export()
    rng = np.random.default_rng(10)
    picks = rng.choice(len(cw), size=min(24, len(cw)), replace=False)
    nonzero = 0
    for i in picks:
        P = cw[i]
        fwd = O.OracleEngine(64, 0.0)
        fwd.set_initial(P[None], [1.0])
        for _ in range(5):  # U P U^dag: gates in circuit order, each conjugated with -theta
            for words, cs, sn in layer:
                fwd.apply_gate(words, cs, -sn)
        bw, bc = fwd.export()
        want = math.fsum(float(x) * amap.get(tuple(int(v) for v in k), 0.0) for k, x in zip(bw, bc))
        got = eng.coefficient(pp.PauliString.from_words([int(v) for v in P]))
        assert abs(got - want) <= 1e-12, (i, got, want)
        nonzero += abs(want) > 1e-9
    assert nonzero >= 8, "sampled keys should mostly be live strings"


def test_regroup_table_overflow_retries(pp, O, monkeypatch):
    """A regroup whose hash table is far too small (PP_TINY_TABLE: 1024 slots
    for 7e6 records) gives up probing early (k_insert's probe cap and overflow
    flag), retries with tables 4x larger, and ends with the same operator:
    config 0 to t = 9, ledgers and sum c^2 against the run with the planned
    table."""
    circ = pp.build_kicked_ising(chain_geometry(pp), 0.3, "-0.5pi", 9)
    init = O.site_word(32, 3)[None]

    def run():
        eng = pp.Engine(64, 0.0)
        eng.set_initial(init, np.array([1.0]))
        rows = eng.run_circuit(circ)
        return [{k: v for k, v in r.items() if k != "wall_ms_per_gate"} for r in rows], eng.norm2()

    ref_rows, ref_norm = run()
    monkeypatch.setenv("PP_TINY_TABLE", "1")
    rows, norm = run()
    assert rows == ref_rows
    assert abs(norm - ref_norm) < 1e-12  # (summed in group order, which follows the table's slot order)
    assert rows[-1]["term_count"] == 81662152
