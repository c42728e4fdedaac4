"""Parity of the CUDA path (through the C-ABI / pybind engine) against the
oracle restatement (oracle/pp_oracle.c), bit-exact for string sets and
coefficients (BASELINE.json north_star tolerance
1e-12 relative applies to <Z>, which is summed in a different order)."""
import math

import numpy as np
import pytest

from conftest import assert_same_terms, gate_tuples

pytestmark = pytest.mark.gpu


def rel_close(a, b, tol=1e-12):
    return abs(a - b) <= tol * max(1.0, abs(b))


def random_words(rng, n):
    w = np.zeros(4, np.uint64)
    for site in range(n):
        w[site // 32] |= np.uint64(int(rng.integers(4))) << np.uint64(2 * (site % 32))
    return w


def run_both(pp, O, n, layers, initial, eps=0.0, cadence="gate", steps=None, check_each=True, fuse=True):
    """layers: list of lists of product Gates (forward order)."""
    words = np.stack([w for w, _ in initial]).astype(np.uint64)
    coeffs = np.array([c for _, c in initial], np.float64)
    eng = pp.Engine(n, eps, cadence, fuse_clifford=fuse)
    eng.set_initial(words, coeffs)
    ora = O.OracleEngine(n, eps, 1 if cadence == "layer" else 0)
    ora.set_initial(words, coeffs)
    circ_layers = layers
    L = len(circ_layers)
    for t in range(1, L + 1):
        layer = circ_layers[L - t]
        eng.apply_gates(list(reversed(layer)))
        for g in reversed(gate_tuples(layer)):
            ora.apply_gate(*g)
        if cadence == "layer":
            eng.truncate_now()
            ora.truncate_now()
        ctr = eng.take_counters()
        octr = ora.take_counters()
        if check_each or t == L:
            w, c = eng.export()
            ow, oc = ora.export()
            assert_same_terms(w, c, ow, oc, f"layer {t}")
            assert eng.term_count() == ora.term_count()
            assert rel_close(eng.expectation_zero_state(), ora.expectation())
            assert eng.global_max() == ora.global_max()
            assert ctr["records_sent"] == octr["records_sent"], (ctr, octr)
            assert ctr["removed"] == octr["removed"], (ctr, octr)
            assert ctr["batches_sent"] == octr["batches_sent"], (ctr, octr)
    return eng, ora


def test_single_qubit_rotation_signs(pp, O):
    # test_engine.cpp:77-91: X under Z(theta) -> cos X, record (Y, -sin)
    theta = 0.81
    eng = pp.Engine(1, 0.0)
    eng.set_initial(O.site_word(0, 1)[None], np.array([1.0]))
    g = pp.Gate(pp.PauliString("Z0", 1), theta)
    eng.apply_gate(g)
    assert eng.coefficient(pp.PauliString("X0", 1)) == math.cos(theta) * 1.0
    assert eng.coefficient(pp.PauliString("Y0", 1)) == -math.sin(theta) * 1.0
    assert eng.term_count() == 2


def test_rx_signs_match_oracle(pp, O):
    # Rx on Z and Y: c'_Y = cos c_Y + sin c_Z ; c'_Z = cos c_Z - sin c_Y
    for init in (["Z0"], ["Y0"], ["Z0", "Y0"]):
        terms = [(np.asarray(pp.PauliString(l, 1).words), 0.5 + i) for i, l in enumerate(init)]
        layers = [[pp.Gate(pp.PauliString("X0", 1), 0.3)]]
        run_both(pp, O, 1, layers, terms)


def test_commuting_and_theta_zero(pp, O):
    # test_engine.cpp:93-120
    terms = [(np.asarray(pp.PauliString("Z2 Z0", 3).words), 0.5), (np.asarray(pp.PauliString("Z1", 3).words), -0.25)]
    run_both(pp, O, 3, [[pp.Gate(pp.PauliString("Z2", 3), 1.1)]], terms)
    run_both(pp, O, 3, [[pp.Gate(pp.PauliString("X0", 3), 0.0)]], terms)
    run_both(pp, O, 3, [[pp.Gate(pp.PauliString("X1", 3), "0.5pi")]], terms)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("eps,cadence", [(0.0, "gate"), (1e-3, "gate"), (1e-2, "layer")])
def test_random_circuits(pp, O, seed, eps, cadence):
    # test_engine.cpp:148-175 / acceptance criterion 3 (random generators of
    # any weight, radian angles in [-3, 3])
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 11))
    layers = []
    for _ in range(int(rng.integers(1, 4))):
        layer = []
        for _ in range(int(rng.integers(1, 8))):
            layer.append(pp.Gate(pp.PauliString.from_words(random_words(rng, n)), float(rng.uniform(-3, 3))))
        layers.append(layer)
    site = int(rng.integers(n))
    run_both(pp, O, n, layers, [(O.site_word(site, 3), 1.0)], eps, cadence)


@pytest.mark.parametrize("seed", range(6))
def test_random_x_and_zz_circuits_many_terms(pp, O, seed):
    # kicked-Ising-like gates (Rx + Rzz, some Clifford) on a random initial sum
    rng = np.random.default_rng(77 + seed)
    n = [5, 12, 40, 64, 65, 127][seed]
    init = []
    for _ in range(60):  # low-weight strings so the exact growth stays small
        w = np.zeros(4, np.uint64)
        for site in rng.choice(n, size=min(n, 3), replace=False):
            w[site // 32] |= np.uint64(int(rng.integers(1, 4))) << np.uint64(2 * (site % 32))
        init.append((w, float(rng.uniform(-1, 1))))
    layer = []
    for q in range(n):
        layer.append(pp.Gate(pp.PauliString(f"X{q}", n), float(rng.uniform(-3, 3))))
    for q in range(n - 1):
        ang = "-0.5pi" if rng.random() < 0.7 else float(rng.uniform(-3, 3))
        layer.append(pp.Gate(pp.PauliString(f"Z{q} Z{q + 1}", n), ang))
    run_both(pp, O, n, [layer], init, 1e-3)


def test_duplicate_and_zero_initial_terms(pp, O):
    n = 4
    a = np.asarray(pp.PauliString("Z0 X1", n).words)
    b = np.asarray(pp.PauliString("Y2", n).words)
    init = [(a, 0.5), (b, 0.0), (a, 0.25), (b, 1e-30), (a, -0.75)]
    layers = [[pp.Gate(pp.PauliString("X0", n), 0.4), pp.Gate(pp.PauliString("Z1 Z2", n), 0.7)]]
    for cad in ("gate", "layer"):
        run_both(pp, O, n, layers, init, 0.0, cad)


def test_identity_generator_and_empty_operator(pp, O):
    n = 3
    layers = [[pp.Gate(pp.PauliString("III", n), 0.5), pp.Gate(pp.PauliString("X1", n), 0.5)]]
    run_both(pp, O, n, layers, [(O.site_word(1, 3), 1.0)])
    eng = pp.Engine(n, 0.0)
    eng.set_initial(np.zeros((0, 4), np.uint64), np.zeros(0))
    eng.apply_gate(layers[0][1])
    assert eng.term_count() == 0
    assert eng.expectation_zero_state() == 0.0


def _kicked(pp, geom, thx, layers):
    return pp.build_kicked_ising(geom, thx, "-0.5pi", layers)


def test_heavy_hex_config1_bitexact(pp, O):
    # BASELINE config 1: theta_h = pi/4, eps0 = 0, Z62, 5 steps (2,146,372 strings)
    geom = pp.heavy_hex_127()
    circ = _kicked(pp, geom, "0.25pi", 5)
    eng, ora = run_both(pp, O, 127, list(circ.layers), [(O.site_word(62, 3), 1.0)], 0.0, "gate")
    assert eng.term_count() == 2146372


def test_table1_rows(pp, O):
    # PAPER.md Table I / acceptance_main.cpp:99-109
    geom = pp.heavy_hex_127()
    exact = [-0.95105651629515, 0.90450849718747, -0.9423841865631, 0.97436799430396, -0.95315824248965]
    tol = [1e-11, 1e-11, 1e-11, 1e-10, 1e-10]
    eng = pp.Engine(127, 0.0)
    eng.set_initial(O.site_word(62, 3)[None], np.array([1.0]))
    rows = eng.run_circuit(_kicked(pp, geom, "0.9pi", 5))
    for r, v, t in zip(rows, exact, tol):
        assert abs(r["observable"] - v) < t
    eng = pp.Engine(127, 1e-5)
    eng.set_initial(O.site_word(62, 3)[None], np.array([1.0]))
    rows = eng.run_circuit(_kicked(pp, geom, "0.9pi", 5))
    assert abs(rows[3]["observable"] - 0.97438562148434) < 1e-9
    assert abs(rows[4]["observable"] - -0.95311531321393) < 1e-9


def test_clifford_regimes(pp, O):
    # acceptance_main.cpp:417-453: theta_x = 0 and pi/2 keep |O| = 1
    geom = pp.heavy_hex_127()
    for thx in ("0pi", "0.5pi"):
        eng = pp.Engine(127, 0.0)
        eng.set_initial(O.site_word(62, 3)[None], np.array([1.0]))
        rows = eng.run_circuit(_kicked(pp, geom, thx, 20))
        assert all(r["term_count"] == 1 for r in rows)
        if thx == "0pi":
            assert all(r["observable"] == 1.0 for r in rows)


def test_chain_config0_bitexact(pp, O):
    # BASELINE config 0 prefix: n = 64 chain, theta_h = 0.3 rad, eps0 = 0
    text = "\n".join(f"{i} {i + 1} {i % 2}" for i in range(63))
    geom = pp.load_geometry(text)
    circ = pp.build_kicked_ising(geom, 0.3, "-0.5pi", 7)
    eng, _ = run_both(pp, O, 64, list(circ.layers), [(O.site_word(32, 3), 1.0)], 0.0, "gate", check_each=False)
    assert eng.term_count() == 613470


def test_truncated_heavy_hex_bitexact(pp, O):
    geom = pp.heavy_hex_127()
    circ = _kicked(pp, geom, "0.25pi", 7)
    run_both(pp, O, 127, list(circ.layers), [(O.site_word(62, 3), 1.0)], 1e-4, "gate", check_each=True)


def test_non_clifford_zz_config4_shape(pp, O):
    # BASELINE config 4 shape: theta_J = -pi/2 + 0.2 (Rzz branches), sum Z_i / 127
    geom = pp.heavy_hex_127()
    circ = pp.build_kicked_ising(geom, 0.4, -math.pi / 2 + 0.2, 3)
    init = [(O.site_word(q, 3), 1.0 / 127) for q in range(127)]
    run_both(pp, O, 127, list(circ.layers), init, 1e-4, "gate")


def test_budget_and_nan(pp, O):
    geom = pp.heavy_hex_127()
    with pytest.raises(pp.ResourceLimitError):
        pp.simulate(_kicked(pp, geom, "0.25pi", 6), observable="Z62", max_terms=100)
    eng = pp.Engine(2, 0.0)
    eng.set_initial(O.site_word(0, 3)[None], np.array([math.inf]))
    with pytest.raises(pp.NumericalError):
        eng.apply_gate(pp.Gate(pp.PauliString("X0", 2), 0.3))


@pytest.mark.parametrize("eps,limit", [(0.0, 1000), (1e-3, 200), (0.0, 40)])
def test_budget_error_fires_where_the_reference_fires(pp, O, eps, limit):
    """check_budget (engine.cpp:266-275): the error comes after the same gate
    of the same layer with the same |O| (counted before that gate's
    truncation) as in the oracle, through run_circuit (fused Clifford runs,
    Rx runs) and gate by gate."""
    import re

    geom = pp.heavy_hex_127()
    circ = _kicked(pp, geom, "0.3pi", 6)
    init = O.site_word(62, 3)[None]
    ora = O.OracleEngine(127, eps, max_terms=limit)
    ora.set_initial(init, [1.0])
    expect = None
    L = len(circ.layers)
    for t in range(1, L + 1):
        for k, g in enumerate(reversed(list(circ.layers[L - t]))):
            try:
                ora.apply_gate(np.asarray(g.generator.words), g.cos_theta, g.sin_theta)
            except O.OracleError:
                expect = (t, ora.take_counters()["gates"], ora.term_count())
                break
        if expect:
            break
    assert expect is not None, "the budget must be exceeded in this circuit"
    for per_gate in (False, True):
        eng = pp.Engine(127, eps, "gate", max_terms=limit)
        eng.set_initial(init, np.array([1.0]))
        with pytest.raises(pp.ResourceLimitError) as err:
            if per_gate:
                for t in range(1, L + 1):
                    eng.set_layer_context(t)
                    for g in reversed(list(circ.layers[L - t])):
                        eng.apply_gate(g)
            else:
                eng.run_circuit(circ)
        m = re.search(r"\|O\|=(\d+) exceeds max_terms=(\d+) at layer (\d+), gate (\d+)", str(err.value))
        assert m, str(err.value)
        assert (int(m.group(3)), int(m.group(4)), int(m.group(1))) == expect, (str(err.value), expect, per_gate)
        assert int(m.group(2)) == limit


def test_simulate_reference_smoke_values(pp):
    # tests/python/test_smoke.py:59-66 of the reference
    geom = pp.heavy_hex_127()
    rows = pp.simulate(pp.build_kicked_ising(geom, "0.9pi", "-0.5pi", layers=1), observable="Z62", workers=2)
    assert len(rows) == 1
    assert rows[0]["observable"] == pytest.approx(math.cos(0.9 * math.pi), abs=1e-12)
    assert rows[0]["term_count"] == 2


def test_fusion_matches_unfused(pp, O):
    geom = pp.heavy_hex_127()
    circ = _kicked(pp, geom, "0.25pi", 4)
    a = pp.Engine(127, 0.0, fuse_clifford=True)
    b = pp.Engine(127, 0.0, fuse_clifford=False)
    for e in (a, b):
        e.set_initial(O.site_word(62, 3)[None], np.array([1.0]))
    ra, rb = a.run_circuit(circ), b.run_circuit(circ)
    wa, ca = a.export()
    wb, cb = b.export()
    ora = O.OracleEngine(127, 0.0)
    ora.set_initial(O.site_word(62, 3)[None], [1.0])
    ora.run_layers([(np.asarray(g.generator.words), g.cos_theta, g.sin_theta) for g in circ.layers[0]], 4)
    ow, oc = ora.export()
    assert_same_terms(wa, ca, ow, oc, "fused vs oracle")
    assert_same_terms(wb, cb, ow, oc, "unfused vs oracle")
    for x, y in zip(ra, rb):
        for k in ("term_count", "removed", "records_sent", "batches_sent"):
            assert x[k] == y[k], (k, x, y)


@pytest.mark.parametrize("mode", ["default", "tight_arena"])
def test_speculative_sublayer_is_exact(pp, O, monkeypatch, mode):
    # the fused run for epsilon0 > 0 (the default: predicted thresholds,
    # verified and rolled back on mismatch, intermediate versions in the CTAs'
    # scratch) must give the per-gate result bit for bit, also when the arena
    # overflows inside a run (PP_TIGHT_ARENA)
    monkeypatch.delenv("PP_NO_SPECULATE", raising=False)
    if mode == "tight_arena":
        monkeypatch.setenv("PP_TIGHT_ARENA", "1")
    geom = pp.heavy_hex_127()
    for thx, eps in (("0.25pi", 1e-4), (0.3, 1e-5)):
        circ = _kicked(pp, geom, thx, 6)
        run_both(pp, O, 127, list(circ.layers), [(O.site_word(62, 3), 1.0)], eps, "gate", check_each=True)


@pytest.mark.parametrize("mode", ["eager", "deferred", "deferred_tight"])
def test_deferred_truncation_is_exact(pp, O, monkeypatch, mode):
    """Per-gate truncation applied lazily (k_thresh/k_flush, the default for
    epsilon0 > 0) equals the eager per-gate compaction and the oracle: string
    sets, coefficient bits, records and removed counts per layer, also when
    the arena overflows mid-run and the run resumes (PP_TIGHT_ARENA)."""
    monkeypatch.setenv("PP_NO_SPECULATE", "1")  # the per-gate launches
    if mode == "eager":
        monkeypatch.setenv("PP_EAGER_TRUNCATION", "1")
    if mode == "deferred_tight":
        monkeypatch.setenv("PP_TIGHT_ARENA", "1")
    geom = pp.heavy_hex_127()
    for thx, eps in (("0.25pi", 1e-4), (0.3, 1e-5), ("0.9pi", 3e-3)):
        circ = _kicked(pp, geom, thx, 6)
        run_both(pp, O, 127, list(circ.layers), [(O.site_word(62, 3), 1.0)], eps, "gate", check_each=True)
    circ = pp.build_kicked_ising(geom, 0.4, -math.pi / 2 + 0.2, 3)
    init = [(O.site_word(q, 3), 1.0 / 127) for q in range(127)]
    run_both(pp, O, 127, list(circ.layers), init, 3e-4, "gate")


@pytest.mark.parametrize("mode", ["per_gate", "dense_tight", "unsorted_fallback", "dense_in_branch_kernel",
                                  "dense_careful", "dense_kernel_tight_maxk"])
def test_sublayer_paths_match_oracle(pp, O, monkeypatch, mode):
    """epsilon0 = 0 Rx runs: the dense sublayer (default: k_dense_sublayer +
    dense_apply, class-major multi-class output) and
    the per-gate segment/stream path (PP_NO_DENSE) both equal the oracle bit
    for bit, also when the arena overflows mid-run and resumes
    (PP_TIGHT_ARENA: dense blocks in global memory and in shared memory), and
    when groups a regroup left unsorted must take the per-gate path."""
    if mode == "per_gate":
        monkeypatch.setenv("PP_NO_DENSE", "1")
    elif mode == "dense_tight":
        monkeypatch.setenv("PP_TIGHT_ARENA", "1")
    elif mode == "dense_in_branch_kernel":
        # the dense path inside k_branch_sublayer instead of k_dense_sublayer
        monkeypatch.setenv("PP_NO_DENSE_KERNEL", "1")
    elif mode == "dense_careful":
        # point-by-point butterflies (dense_bfly) instead of the bookkeeping-free passes
        monkeypatch.setenv("PP_DENSE_CAREFUL", "1")
    elif mode == "dense_kernel_tight_maxk":
        # k_dense_sublayer leaves groups of more than 2 classes to the per-gate
        # pass behind it, with arena overflows and resumes on top
        monkeypatch.setenv("PP_DENSE_MAXK", "2")
        monkeypatch.setenv("PP_TIGHT_ARENA", "1")
    else:
        # multi-class groups leave the dense path after a regroup that skipped
        # its sort: the sublayer defers them, the host sorts, the run resumes
        monkeypatch.setenv("PP_DENSE_MAXK", "1")
    geom = pp.heavy_hex_127()
    circ = _kicked(pp, geom, "0.25pi", 5)
    run_both(pp, O, 127, list(circ.layers), [(O.site_word(62, 3), 1.0)], 0.0, "gate", check_each=True)
    text = "\n".join(f"{i} {i + 1} {i % 2}" for i in range(63))
    circ = pp.build_kicked_ising(pp.load_geometry(text), 0.3, "-0.5pi", 7)
    run_both(pp, O, 64, list(circ.layers), [(O.site_word(32, 3), 1.0)], 0.0, "gate", check_each=True)
    # heavy-hex away from pi/4 (no exact cancellations: the bookkeeping-free passes keep their tiles)
    circ = _kicked(pp, geom, 0.37, 4)
    run_both(pp, O, 127, list(circ.layers), [(O.site_word(62, 3), 1.0)], 0.0, "gate", check_each=True)


def test_engine_pool_reuse_is_fresh(pp, O):
    """Released engines are pooled and handed to the next creation with the
    same configuration (pp_create / pp_destroy): the reused engine starts as
    an empty operator with zeroed counters, and a run on it equals the
    oracle bit for bit."""
    import gc

    geom = pp.heavy_hex_127()
    circ = _kicked(pp, geom, "0.25pi", 4)
    a = pp.Engine(127, 0.0)
    a.set_initial(O.site_word(62, 3)[None], np.array([1.0]))
    a.run_circuit(circ)
    del a
    gc.collect()
    b = pp.Engine(127, 0.0)  # the pooled engine
    assert b.term_count() == 0
    assert b.take_counters()["records_sent"] == 0
    del b
    gc.collect()
    # run_both's engine is the pooled one again; a different observable
    run_both(pp, O, 127, list(circ.layers), [(O.site_word(61, 3), 1.0), (O.site_word(63, 1), 0.5)], 0.0, "gate",
             check_each=True)


def test_chain_config0_t8_dense_big_blocks(pp, O):
    """BASELINE config 0 to t = 8 (6,952,660 strings): the last Rx run has
    groups of several x classes with 2^m > one shared-memory tile (the dense
    path's global-memory passes, class-major output and hole compaction) --
    bit-exact against the oracle."""
    text = "\n".join(f"{i} {i + 1} {i % 2}" for i in range(63))
    circ = pp.build_kicked_ising(pp.load_geometry(text), 0.3, "-0.5pi", 8)
    eng, _ = run_both(pp, O, 64, list(circ.layers), [(O.site_word(32, 3), 1.0)], 0.0, "gate", check_each=False)
    assert eng.term_count() == 6952660


@pytest.mark.parametrize("n", [64, 127])
def test_dense_big_and_multiclass_blocks(pp, O, n):
    """Groups built to take every dense sub-path in one Rx layer: several x
    classes with 2^m above a shared-memory tile (global passes, bulk-copied
    tile rows, class-major output), several classes batched through one tile, and one class of
    several strings with 2^m above a tile -- bit-exact against the oracle."""
    rng = np.random.default_rng(n)

    def word(label):
        return np.asarray(pp.PauliString(label, n).words, np.uint64)

    def zs(sites, ys=()):
        return " ".join(("Y" if q in ys else "Z") + str(q) for q in sites)

    base = 40 if n == 64 else 100
    big = list(range(14))                 # m = 14: 2^14 points > one tile
    mid = list(range(base - 20, base - 8))  # m = 12
    init = []
    for j, extra in enumerate([f"X{base}", f"X{base + 1}", f"X{base} X{base + 1}"]):  # K = 3 classes
        init.append((word(zs(big, ys=(j,)) + " " + extra), float(rng.uniform(-1, 1))))
    for a, b in [(0, 0), (0, 1), (1, 0), (1, 1)]:  # K = 4 classes, batched two per tile
        extra = " ".join(s for s, on in ((f"X{base + 2}", a), (f"X{base + 3}", b)) if on)
        init.append((word(zs(mid) + (" " + extra if extra else "")), float(rng.uniform(-1, 1))))
    for ys in [(20,), (21, 22), (23,)]:  # one class, several strings, m = 14
        sites = list(range(16, 30))
        init.append((word(zs(sites, ys=ys)), float(rng.uniform(-1, 1))))
    layer = [pp.Gate(pp.PauliString(f"X{q}", n), float(rng.uniform(-3, 3))) for q in range(n)]
    run_both(pp, O, n, [layer], init, 0.0, "gate", check_each=True)


def test_reinitialised_engine_big_group_then_zz(pp, O):
    """A pooled engine (and a second set_initial on one engine) starts from
    the new operator's group statistics: a z-group of 1024 strings followed by
    a non-Clifford ZZ as the first gate is exact (maxcnt_ was kept
    from the previous operator)."""
    n = 24
    # z = Z on sites 0..9 plus 12, x free on 0..9: 1024 strings in one z-group
    words, coeffs = [], []
    rng = np.random.default_rng(3)
    for xbits in range(1024):
        w = np.zeros(4, np.uint64)
        for q in range(10):
            code = 2 if (xbits >> q) & 1 else 3  # Y (x=1, z=1) or Z (x=0, z=1)
            w[0] |= np.uint64(code) << np.uint64(2 * q)
        w[0] |= np.uint64(3) << np.uint64(24)
        words.append(w)
        coeffs.append(float(rng.uniform(-1, 1)))
    words = np.stack(words)
    coeffs = np.array(coeffs)
    zz = pp.Gate(pp.PauliString("Z0 Z20", n), 0.37)
    rx = pp.Gate(pp.PauliString("X3", n), 0.21)
    for trial in range(3):
        eng = pp.Engine(n, 0.0)
        if trial == 0:  # a used engine re-initialised in place
            eng.set_initial(O.site_word(5, 3)[None], np.array([1.0]))
            eng.apply_gates([rx, zz])
        eng.set_initial(words, coeffs)
        eng.apply_gates([zz, rx, zz])
        ora = O.OracleEngine(n, 0.0)
        ora.set_initial(words, coeffs)
        for g in (zz, rx, zz):
            ora.apply_gate(np.asarray(g.generator.words, np.uint64), g.cos_theta, g.sin_theta)
        w, c = eng.export()
        ow, oc = ora.export()
        assert_same_terms(w, c, ow, oc, f"trial {trial}")
        del eng  # trial 1, 2: the next Engine is the pooled one


def test_tracked_coefficient_and_gate_readout(pp, O):
    """RunOptions readout modes (engine.hpp:203-213): TrackedCoefficient per
    layer and the per-gate on_gate_readout trace, against the oracle."""
    geom = pp.heavy_hex_127()
    circ = _kicked(pp, geom, 0.3, 3)
    z62 = pp.PauliString("Z62", 127)
    tracked = pp.PauliString("Z62 X63", 127)
    eng = pp.Engine(127, 1e-5)
    eng.set_initial(O.site_word(62, 3)[None], np.array([1.0]))
    trace = []
    rows = eng.run_circuit(circ, readout="coefficient", tracked=tracked,
                           on_gate_readout=lambda t, gi, v: trace.append((t, gi, v)))
    ora = O.OracleEngine(127, 1e-5)
    ora.set_initial(O.site_word(62, 3)[None], [1.0])
    tw = np.asarray(tracked.words, np.uint64)
    k = 0
    L = circ.num_layers()
    for t in range(1, L + 1):
        for gi, g in enumerate(reversed(circ.layers[L - t])):
            ora.apply_gate(np.asarray(g.generator.words, np.uint64), g.cos_theta, g.sin_theta)
            tt, tgi, v = trace[k]
            assert (tt, tgi) == (t, gi)
            assert v == ora.coefficient(tw), (t, gi)  # a coefficient is one string's value: bit-exact
            k += 1
        assert rows[t - 1]["observable"] == ora.coefficient(tw)
    assert k == len(trace) == circ.total_gates()
    # the default readout and a tracked Z62 agree with <0|O|0>'s single-string case at t = 0
    e2 = pp.Engine(127, 0.0)
    e2.set_initial(O.site_word(62, 3)[None], np.array([1.0]))
    assert e2.run_circuit(_kicked(pp, geom, "0.5pi", 1), readout="coefficient", tracked=z62)[0]["term_count"] == 1


def test_shards_mirror_the_reference_partition(pp, O):
    """Engine.shards()/shard_sizes() (engine.hpp:161-162): the operator split
    by the reference's block-sum owner map, sizes equal to the reference's own
    shards at the same worker count; PhaseTimers present in the counters."""
    if not O.ref_available():
        pytest.skip("reference library not built")
    geom = pp.heavy_hex_127()
    circ = _kicked(pp, geom, "0.25pi", 4)
    for workers in (1, 4, 7):
        eng = pp.Engine(127, 0.0, workers=workers)
        eng.set_initial(O.site_word(62, 3)[None], np.array([1.0]))
        eng.run_circuit(circ)
        ref = O.RefEngine(127, 0.0, workers=workers, threads=workers)
        ref.set_initial(O.site_word(62, 3)[None], [1.0])
        gates = [(np.asarray(g.generator.words, np.uint64), 0.25 if i < 127 else -0.5, 1)
                 for i, g in enumerate(circ.layers[0])]
        ref.run_circuit(gates, 4)
        assert eng.shard_sizes() == ref.shard_sizes(), workers
        shards = eng.shards()
        assert len(shards) == workers and sum(len(c) for _, c in shards) == eng.term_count()
        spec = pp.PartitionSpec(workers=workers)  # block_size_bits 0: the default k
        for m, (w, c) in enumerate(shards):
            for row in w[:50]:
                assert pp.owner(spec, pp.PauliString.from_words([int(v) for v in row]), 127) == m
    t = eng.take_counters()["timers"]
    assert set(t) == {"generate_ns", "exchange_ns", "apply_ns", "truncate_ns"}
