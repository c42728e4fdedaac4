"""Pins the oracle restatement (oracle/pp_oracle.c) to the reference: every
golden fixture in tests/golden/ was produced by the reference engine itself
(tests/golden/make_golden.py over oracle/_ref).  CPU only."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def ledgers():
    with open(os.path.join(GOLD, "ledgers.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def states():
    return dict(np.load(os.path.join(GOLD, "states.npz")))


@pytest.fixture(scope="module")
def algebra():
    with open(os.path.join(GOLD, "algebra.json")) as f:
        return json.load(f)


def ref_order_layer(O, n, thx, thx_pi, thzz, thzz_pi, geometry):
    """Kicked-Ising layer in the reference's gate order, with the
    restatement's own trig (oracle_angle == circuit.cpp:28-63)."""
    if geometry == "chain":
        edges = [(i, i + 1, i % 2) for i in range(n - 1)]
    else:
        edges = []
        for line in open(os.path.join(GOLD, "heavy_hex_ref_order.txt")):
            if line.startswith("#") or not line.strip():
                continue
            a, b, c = map(int, line.split())
            edges.append((a, b, c))
    cx, sx, _ = O.oracle_angle(thx, thx_pi)
    cz, sz, _ = O.oracle_angle(thzz, thzz_pi)
    gates = [(O.site_word(q, 1), cx, sx) for q in range(n)]
    for col in range(max(e[2] for e in edges) + 1):
        for a, b, c in edges:
            if c == col:
                gates.append((O.site_word(a, 3) | O.site_word(b, 3), cz, sz))
    return gates


CASES = ["config1_pi4_eps0", "table1_0.9pi_eps0", "table1_0.9pi_eps1e-5", "hh_pi4_eps1e-4",
         "hh_0.3rad_eps1e-5_layer", "chain64_0.3rad_eps0", "config4_shape_eps1e-4"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_ledgers_match_reference(O, ledgers, name):
    case = next(c for c in ledgers["cases"] if c["name"] == name)
    layers = min(case["layers"], 5)
    gates = ref_order_layer(O, case["n"], case["theta_x"], case["theta_x_pi"], case["theta_zz"], case["theta_zz_pi"],
                            case["geometry"])
    eng = O.OracleEngine(case["n"], case["epsilon0"], case["cadence"])
    w = np.stack([O.site_word(s, 3) for s, _ in case["init"]])
    eng.set_initial(w, [c for _, c in case["init"]])
    rows = eng.run_layers(gates, layers)
    for got, want in zip(rows, case["rows"][:layers]):
        assert got["term_count"] == want["term_count"]
        assert np.float64(got["global_max"]).view(np.uint64) == want["global_max_bits"]
        assert got["removed"] == want["removed"]
        assert got["records_sent"] == want["records_sent"]
        assert got["batches_sent"] == want["batches_sent"]
        assert abs(got["observable"] - want["observable"]) <= 1e-12 * max(1, abs(want["observable"]))


def test_table1_golden_values(ledgers):
    # PAPER.md Table I (acceptance_main.cpp:99-109) reproduced by the reference run
    exact = [-0.95105651629515, 0.90450849718747, -0.9423841865631, 0.97436799430396, -0.95315824248965]
    case = next(c for c in ledgers["cases"] if c["name"] == "table1_0.9pi_eps0")
    for r, v in zip(case["rows"], exact):
        assert abs(r["observable"] - v) < 1e-10
    case = next(c for c in ledgers["cases"] if c["name"] == "table1_0.9pi_eps1e-5")
    assert abs(case["rows"][3]["observable"] - 0.97438562148434) < 1e-9
    assert abs(case["rows"][4]["observable"] - -0.95311531321393) < 1e-9


@pytest.mark.parametrize("name,n,thx,pi,site,layers", [("config1_t3", 127, 0.25, 1, 62, 3),
                                                       ("chain64_t4", 64, 0.3, 0, 32, 4)])
def test_oracle_states_match_reference(O, states, name, n, thx, pi, site, layers):
    gates = ref_order_layer(O, n, thx, pi, -0.5, 1, "chain" if n == 64 else "hh")
    eng = O.OracleEngine(n, 0.0)
    eng.set_initial(O.site_word(site, 3)[None], [1.0])
    eng.run_layers(gates, layers)
    w, c = eng.export()
    assert (w == states[name + "_words"]).all()
    assert (c.view(np.uint64) == states[name + "_coeff_bits"]).all()


def test_oracle_random_circuits_match_reference(O, ledgers, states):
    # any-weight generators, radian angles (test_engine.cpp:148-175 style)
    for k, rc in enumerate(ledgers["random"]):
        eng = O.OracleEngine(rc["n"], rc["epsilon0"])
        eng.set_initial(O.site_word(rc["site"], 3)[None], [1.0])
        for layer in reversed(rc["layers"]):
            for words, theta in reversed(layer):
                c, s, _ = O.oracle_angle(theta, 0)
                eng.apply_gate(np.array(words, np.uint64), c, s)
        w, c = eng.export()
        assert (w == states[f"random{k}_words"]).all(), k
        assert (c.view(np.uint64) == states[f"random{k}_coeff_bits"]).all(), k


def test_oracle_phase_table_and_angles(O, algebra):
    for a, b, want in algebra["phase_pairs"]:
        assert O.oracle_phase_exponent(O.site_word(0, a), O.site_word(0, b), 1) == want
    for ang in algebra["angles"]:
        c, s, r = O.oracle_angle(ang["value"], ang["pi_units"])
        assert np.float64(c).view(np.uint64) == ang["cos_bits"]
        assert np.float64(s).view(np.uint64) == ang["sin_bits"]


def _symplectic_b(xi, zi, xj, zj):
    """Python restatement of the 4-popcount phase used by the kernels
    (pp_common.cuh phase_mod4)."""
    pc = lambda v: bin(v).count("1")  # noqa: E731
    return (pc(xi & zi) + pc(xj & zj) + 2 * pc(zi & xj) - pc((xi ^ xj) & (zi ^ zj))) % 4


def test_symplectic_phase_identity(O, algebra):
    # exhaustive on one site, random on 128 sites, against the phase table
    for a, b, want in algebra["phase_pairs"]:
        xa, za = O.to_planes(O.site_word(0, a)[None])
        xb, zb = O.to_planes(O.site_word(0, b)[None])
        assert _symplectic_b(int(xa[0, 0]), int(za[0, 0]), int(xb[0, 0]), int(zb[0, 0])) == want
    rng = np.random.default_rng(3)
    for _ in range(300):
        wa = rng.integers(0, 2**63, size=4, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, 4, dtype=np.uint64)
        wb = rng.integers(0, 2**63, size=4, dtype=np.uint64)
        xa, za = O.to_planes(wa[None])
        xb, zb = O.to_planes(wb[None])
        pack = lambda p: int(p[0][0]) | (int(p[0][1]) << 64)  # noqa: E731
        assert _symplectic_b(pack(xa), pack(za), pack(xb), pack(zb)) == O.oracle_phase_exponent(wa, wb, 128)


def test_plane_conversion_round_trip(O):
    rng = np.random.default_rng(5)
    w = rng.integers(0, 2**63, size=(1000, 4), dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, (1000, 4),
                                                                                               dtype=np.uint64)
    x, z = O.to_planes(w)
    assert (O.from_planes(x, z) == w).all()
    # codes: I=00 X=01 Y=10 Z=11 -> (x, z) = (0,0) (1,0) (1,1) (0,1)
    for code, (ex, ez) in zip(range(4), [(0, 0), (1, 0), (1, 1), (0, 1)]):
        x, z = O.to_planes(O.site_word(5, code)[None])
        assert int(x[0][0]) == ex << 5 and int(z[0][0]) == ez << 5


@pytest.mark.parametrize("eps,limit", [(0.0, 1000), (1e-3, 200), (0.0, 40)])
def test_oracle_budget_error_matches_reference(O, eps, limit):
    """check_budget (engine.cpp:266-275): the restatement refuses the same
    gate with the same |O| as the reference engine (compiled from its sources,
    oracle/_ref); the reference's message carries both."""
    import re

    if not O.ref_available():
        pytest.skip("oracle/_ref is not built (needs /root/reference)")
    layer = ref_order_layer(O, 127, 0.3, 1, -0.5, 1, "heavy_hex")
    ref = O.RefEngine(127, eps, max_terms=limit)
    ora = O.OracleEngine(127, eps, max_terms=limit)
    init = O.site_word(62, 3)[None]
    ref.set_initial(init, [1.0])
    ora.set_initial(init, [1.0])
    ref_gates = [(w, 0.3 if c != 0.0 and abs(s) != 1.0 else -0.5, 1) for (w, c, s) in layer]
    with pytest.raises(O.OracleError) as err:
        for _ in range(8):
            ref.run_circuit(ref_gates)
    m = re.search(r"\|O\|=(\d+) exceeds max_terms=(\d+) at layer (\d+), gate (\d+)", str(err.value))
    assert m, str(err.value)
    got = None
    for _ in range(8):
        for w, c, s in reversed(layer):
            try:
                ora.apply_gate(w, c, s)
            except O.OracleError:
                got = (ora.take_counters()["gates"], ora.term_count())
                break
        if got:
            break
    assert got == (int(m.group(4)), int(m.group(1))), (str(err.value), got)
