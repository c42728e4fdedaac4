"""Device density histogram and checkpoint/resume on the GPU engine.

* pp_density_histogram counts equal the oracle's exactly and the TSV equals
  the reference's bytes (tests/golden/histograms.json).
* run_circuit's per-layer outputs follow runner.cpp:173-183
  (histogram_t<t>.tsv, checkpoint_t<t>/{manifest.json, shard_0.txt}).
* Resume: checkpoint at layer k, load into a fresh engine, continue with
  start_layer=k -> identical strings, coefficient bits and ledger rows as the
  uninterrupted run (the reference writes checkpoints but cannot resume).
* A checkpoint in the reference's own layout loads and continues bit-exact
  against the oracle continuing from the same state."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT, assert_same_terms, gate_tuples
from test_diagnostics_cpu import _reference_layout_checkpoint, histos, ledgers, oracle_state  # noqa: F401
from test_oracle_pins import ref_order_layer

pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden")


def _engine_from_oracle(pp, ora, n, eps, cadence="gate"):
    w, c = ora.export()
    e = pp.Engine(n, eps, cadence)
    e.set_initial(w, c)
    return e


def test_device_histogram_counts_and_tsv(pp, O, histos, ledgers):  # noqa: F811
    done = {}
    for h in histos:
        key = (h["case"], h["layers"])
        if key not in done:
            ora = oracle_state(O, ledgers, *key)
            n = 64 if key[0] == "chain64_t4" else 127
            eps = h["epsilon0"]
            done[key] = (ora, _engine_from_oracle(pp, ora, n, eps))
        ora, eng = done[key]
        # x = c / the oracle's (== reference's) global max after the run
        got = eng.density_histogram(h["bins"], h["epsilon0"], ora.global_max())
        pos, neg = ora.density_histogram(h["bins"], h["epsilon0"])
        assert got["positive_counts"] == pos.tolist(), key
        assert got["negative_counts"] == neg.tolist(), key
        assert got["tsv"] == h["tsv"], key


def test_device_histogram_large_state(pp, O):
    """3e5-string state: device counts equal the oracle's bin for bin."""
    geom = pp.load_geometry("\n".join(f"{i} {i + 1} {i % 2}" for i in range(63)))
    circ = pp.build_kicked_ising(geom, 0.3, "-0.5pi", 6)
    eng = pp.Engine(64, 0.0)
    eng.set_initial(O.site_word(32, 3)[None], [1.0])
    eng.run_circuit(circ)
    w, c = eng.export()
    ora = O.OracleEngine(64, 0.0)
    ora.set_initial(w, c)
    g = float(np.abs(c).max())
    for bins, eps in [(64, 0.0), (4096, 1e-9), (1, 0.0)]:
        got = eng.density_histogram(bins, eps, g)
        pos, neg = ora.density_histogram(bins, eps, g)
        assert got["positive_counts"] == pos.tolist() and got["negative_counts"] == neg.tolist(), bins
        assert got["total_terms"] == len(c)


def _ref_bin(ax, bins, lower):
    """sparse_operator.cpp:177-186 with the host libm (Python's math.log is
    the same glibc log the reference calls)."""
    import math
    if ax <= lower:
        return 0
    if ax >= 1.0:
        return bins - 1
    return min(max(int(bins * (1.0 - math.log(ax) / math.log(lower))), 0), bins - 1)


@pytest.mark.parametrize("bins,eps", [(64, 0.0), (37, 1e-5), (1000, 1e-12)])
def test_device_histogram_bin_edges_exact(pp, O, bins, eps):
    """Values one ulp either side of every bin boundary land in the
    reference's bin: the kernel compares against host-computed edges, so a
    device-vs-glibc log difference cannot move a string."""
    import math
    lower = max(eps, 1e-16)
    vals = []
    for b in range(1, bins):
        # the nominal boundary, then walk to the exact first double of bin b
        x = math.exp(math.log(lower) * (1.0 - b / bins))
        for _ in range(64):
            if _ref_bin(x, bins, lower) >= b and _ref_bin(math.nextafter(x, 0.0), bins, lower) < b:
                break
            x = math.nextafter(x, 0.0) if _ref_bin(x, bins, lower) >= b else math.nextafter(x, 2.0)
        vals += [math.nextafter(x, 0.0), x, math.nextafter(x, 2.0)]
    vals += [lower, math.nextafter(lower, 2.0), 1.0, math.nextafter(1.0, 0.0)]
    n = len(vals)
    sites = 12  # distinct strings: x patterns over 12 sites (4^12 > n)
    words = np.zeros((n, 4), np.uint64)
    for i in range(n):
        v, w = i + 1, 0
        for s in range(sites):
            w |= (v % 4) << (2 * s)
            v //= 4
        words[i, 0] = w
    coeffs = np.array([v if i % 2 else -v for i, v in enumerate(vals)])
    e = pp.Engine(sites, 0.0)
    e.set_initial(words, coeffs)
    got = e.density_histogram(bins, eps, 1.0)
    pos = [0] * bins
    neg = [0] * bins
    for c in coeffs:
        (neg if c < 0 else pos)[_ref_bin(abs(c), bins, lower)] += 1
    assert got["positive_counts"] == pos and got["negative_counts"] == neg


def test_device_histogram_rejects_zero_max(pp, O):
    e = pp.Engine(2, 0.0)
    e.set_initial(O.site_word(0, 3)[None], [1.0])
    with pytest.raises(ValueError):
        e.density_histogram(4, 0.0, 0.0)
    with pytest.raises(ValueError):
        e.density_histogram(0, 0.0, 1.0)


def test_early_layer_stays_peaked(pp):
    """test_engine.cpp:355-376: one layer at 0.1 pi has <= 4 occupied bins."""
    circ = pp.build_kicked_ising(pp.heavy_hex_127(), "0.1pi", "-0.5pi", 1)
    e = pp.Engine(127, 0.0)
    e.set_initial(np.asarray(pp.parse_pauli_label("Z62", 127).words, np.uint64)[None], [1.0])
    e.run_circuit(circ)
    assert e.term_count() <= 16
    h = e.density_histogram(32, 0.0)
    assert sum((p > 0) + (q > 0) for p, q in zip(h["positive"], h["negative"])) <= 4


def _z62(pp):
    return np.asarray(pp.parse_pauli_label("Z62", 127).words, np.uint64)[None]


@pytest.mark.parametrize("binary", [False, True])
@pytest.mark.parametrize("eps,cadence", [(1e-4, "gate"), (1e-3, "layer"), (0.0, "gate")])
def test_checkpoint_resume_is_bit_exact(pp, tmp_path, binary, eps, cadence):
    L, k = (5, 2) if eps > 0 else (4, 2)
    circ = pp.build_kicked_ising(pp.heavy_hex_127(), 0.3, "-0.5pi", L)
    full = pp.Engine(127, eps, cadence)
    full.set_initial(_z62(pp), [1.0])
    rows_full = full.run_circuit(circ, out_dir=str(tmp_path), histogram_bins=8, checkpoint_every=k,
                                 binary_checkpoint=binary)
    fw, fc = full.export()
    ck = tmp_path / f"checkpoint_t{k}"
    man = json.load(open(ck / "manifest.json"))
    assert man["layer"] == k and man["qubits"] == 127 and man["files"][0]["terms"] == rows_full[k - 1]["term_count"]
    for t in range(1, L + 1):
        assert (tmp_path / f"histogram_t{t}.tsv").exists()
    resumed = pp.Engine(127, eps, cadence)
    assert resumed.load_checkpoint(str(ck)) == k
    assert resumed.term_count() == rows_full[k - 1]["term_count"]
    rows = resumed.run_circuit(circ, start_layer=k)
    assert [r["t"] for r in rows] == list(range(k + 1, L + 1))
    rw, rc = resumed.export()
    assert_same_terms(rw, rc, fw, fc, f"resume eps={eps} {cadence} binary={binary}")
    for a, b in zip(rows, rows_full[k:]):
        assert a["term_count"] == b["term_count"] and a["removed"] == b["removed"]
        assert a["observable"] == b["observable"] and a["global_max"] == b["global_max"]


def test_simulate_resume_from(pp, tmp_path):
    circ = pp.build_kicked_ising(pp.heavy_hex_127(), 0.3, "-0.5pi", 4)
    full = pp.simulate(circ, observable="Z62", epsilon0=1e-4, out_dir=str(tmp_path), checkpoint_every=3,
                       histogram_bins=16)
    rows = pp.simulate(circ, observable="Z62", epsilon0=1e-4, resume_from=str(tmp_path / "checkpoint_t3"))
    assert len(rows) == 1 and rows[0]["t"] == 4
    assert rows[0]["observable"] == full[3]["observable"] and rows[0]["term_count"] == full[3]["term_count"]
    tsv = (tmp_path / "histogram_t4.tsv").read_text()
    assert tsv.count("\n") == 1 + 2 * 16


def test_reference_layout_checkpoint_continues_like_oracle(pp, O, tmp_path):
    text = open(os.path.join(GOLD, "dump_chain64_t4.txt")).read()
    _reference_layout_checkpoint(str(tmp_path), text, 4, 64, 0.0)
    geom = pp.load_geometry("\n".join(f"{i} {i + 1} {i % 2}" for i in range(63)))
    circ = pp.build_kicked_ising(geom, 0.3, "-0.5pi", 5)
    e = pp.Engine(64, 0.0)
    assert e.load_checkpoint(str(tmp_path)) == 4
    e.run_circuit(circ, start_layer=4)
    ck = pp.read_checkpoint(str(tmp_path))
    ora = O.OracleEngine(64, 0.0)
    ora.set_initial(ck["words"], ck["coeffs"])
    for g in reversed(gate_tuples(circ.layers[0])):
        ora.apply_gate(*g)
    w, c = e.export()
    ow, oc = ora.export()
    assert_same_terms(w, c, ow, oc, "reference checkpoint + 1 layer")


def test_start_layer_out_of_range(pp):
    circ = pp.build_kicked_ising(pp.heavy_hex_127(), 0.3, "-0.5pi", 2)
    e = pp.Engine(127, 0.0)
    e.set_initial(_z62(pp), [1.0])
    with pytest.raises(ValueError):
        e.run_circuit(circ, start_layer=3)
    assert e.run_circuit(circ, start_layer=2) == []
