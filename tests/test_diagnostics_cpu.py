"""Density histogram and checkpoint formats on CPU.

* The oracle's per-bin counts (oracle/pp_oracle.c ppo_density_histogram,
  restating sparse_operator.cpp:150-197), normalized and formatted by the
  product's host code (histogram_from_counts / to_tsv), reproduce the
  reference's own TSV byte for byte (tests/golden/histograms.json).
* The shard dump format (sparse_operator.cpp:99-122) and checkpoint
  directories (runner.cpp:52-77) round-trip through the product's readers,
  including a checkpoint laid out exactly as the reference writes one.
The engine-side (GPU) halves are in tests/test_gpu_diagnostics.py."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT
from test_oracle_pins import ref_order_layer

GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def histos():
    with open(os.path.join(GOLD, "histograms.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def ledgers():
    with open(os.path.join(GOLD, "ledgers.json")) as f:
        return json.load(f)


def oracle_state(O, ledgers, name, layers):
    if name == "chain64_t4":
        gates = ref_order_layer(O, 64, 0.3, 0, -0.5, 1, "chain")
        eng = O.OracleEngine(64, 0.0)
        eng.set_initial(O.site_word(32, 3)[None], [1.0])
        eng.run_layers(gates, layers)
        return eng
    case = next(c for c in ledgers["cases"] if c["name"] == name)
    gates = ref_order_layer(O, case["n"], case["theta_x"], case["theta_x_pi"], case["theta_zz"],
                            case["theta_zz_pi"], case["geometry"])
    eng = O.OracleEngine(case["n"], case["epsilon0"], case["cadence"])
    eng.set_initial(np.stack([O.site_word(s, 3) for s, _ in case["init"]]), [c for _, c in case["init"]])
    eng.run_layers(gates, layers)
    return eng


def test_histogram_tsv_matches_reference_bytes(pp, O, histos, ledgers):
    states = {}
    for h in histos:
        key = (h["case"], h["layers"])
        if key not in states:
            states[key] = oracle_state(O, ledgers, *key)
        pos, neg = states[key].density_histogram(h["bins"], h["epsilon0"])
        got = pp.histogram_from_counts(h["bins"], h["epsilon0"], pos.tolist(), neg.tolist())
        assert got["tsv"] == h["tsv"], f"{key} bins={h['bins']}"
        assert got["total_terms"] == states[key].term_count()


# mirrors of the reference's unit tests (test_sparse_operator.cpp:152-197)
def _counts(O, n, terms, bins, eps, gmax):
    e = O.OracleEngine(n, 0.0)
    e.set_initial(np.stack([w for w, _ in terms]), [c for _, c in terms])
    return e.density_histogram(bins, eps, gmax)


def test_histogram_single_term_top_bin(pp, O):
    pos, neg = _counts(O, 2, [(O.site_word(0, 3), 1.0)], 10, 1e-6, 1.0)
    h = pp.histogram_from_counts(10, 1e-6, pos.tolist(), neg.tolist())
    assert h["positive"][-1] == 1.0 and sum(h["positive"]) + sum(h["negative"]) == 1.0


def test_histogram_symmetric_pair_splits_by_sign(pp, O):
    pos, neg = _counts(O, 2, [(O.site_word(0, 3), 1.0), (O.site_word(0, 1), -1.0)], 8, 1e-6, 1.0)
    h = pp.histogram_from_counts(8, 1e-6, pos.tolist(), neg.tolist())
    assert h["positive"][-1] == 0.5 and h["negative"][-1] == 0.5


def test_histogram_edges_and_shape(pp):
    h = pp.histogram_from_counts(4, 1e-4, [0, 1, 0, 2], [1, 0, 0, 0])
    assert h["bin_edges"][0] == pytest.approx(1e-4) and h["bin_edges"][-1] == 1.0
    assert h["tsv"].startswith("bin_low\tbin_high\tsign\tnormalized_count\n")
    assert h["tsv"].count("\n") == 1 + 2 * 4
    assert h["total_terms"] == 4
    with pytest.raises(Exception):
        pp.histogram_from_counts(0, 1e-4, [], [])


def test_oracle_histogram_rejects_zero_max(O):
    e = O.OracleEngine(2, 0.0)
    e.set_initial(O.site_word(0, 3)[None], [1.0])
    with pytest.raises(O.OracleError):
        e.density_histogram(4, 0.0, 0.0)


def _golden_state():
    st = np.load(os.path.join(GOLD, "states.npz"))
    return st["chain64_t4_words"], st["chain64_t4_coeff_bits"]


def test_load_dump_reads_reference_dump(pp):
    text = open(os.path.join(GOLD, "dump_chain64_t4.txt")).read()
    w, c = pp.load_dump(text, 64)
    gw, gc = _golden_state()
    assert (w == gw).all() and (c.view(np.uint64) == gc).all()


def test_dump_operator_lines_match_reference(pp):
    gw, gc = _golden_state()
    ours = pp.dump_operator(gw, gc.view(np.float64), 64)
    ref = open(os.path.join(GOLD, "dump_chain64_t4.txt")).read()
    assert sorted(ours.splitlines()) == sorted(ref.splitlines())


def test_load_dump_rejects_malformed_line(pp):
    with pytest.raises(ValueError):
        pp.load_dump("zz\n", 4)
    with pytest.raises(ValueError):
        pp.load_dump("0x3 \n", 4)


def _reference_layout_checkpoint(d, text, layer, n, eps):
    """A checkpoint directory as runner.cpp:52-77 writes it (two workers,
    nlohmann dump(2) manifest)."""
    lines = text.splitlines(keepends=True)
    parts = [lines[0::2], lines[1::2]]
    files = []
    for m, part in enumerate(parts):
        name = f"shard_{m}.txt"
        with open(os.path.join(d, name), "w") as f:
            f.writelines(part)
        files.append({"path": name, "terms": len(part), "worker": m})
    manifest = {"block_size_bits": 1, "epsilon0": eps, "files": files, "layer": layer,
                "perturbation_hash": "splitmix64-finalizer-word-fold", "perturbation_s": 1,
                "qubits": n, "schema": 1, "workers": 2}
    with open(os.path.join(d, "manifest.json"), "w") as f:
        f.write(json.dumps(manifest, indent=2, sort_keys=True) + "\n")


def test_read_reference_layout_checkpoint(pp, tmp_path):
    text = open(os.path.join(GOLD, "dump_chain64_t4.txt")).read()
    _reference_layout_checkpoint(str(tmp_path), text, 4, 64, 0.0)
    ck = pp.read_checkpoint(str(tmp_path))
    gw, gc = _golden_state()
    assert ck["layer"] == 4 and ck["qubits"] == 64
    assert (ck["words"] == gw).all() and (ck["coeffs"].view(np.uint64) == gc).all()


@pytest.mark.parametrize("binary", [False, True])
def test_checkpoint_files_round_trip(pp, tmp_path, binary):
    gw, gc = _golden_state()
    c = gc.view(np.float64)
    half = len(c) // 2
    ext = "ppb" if binary else "txt"
    files = []
    for m, sl in enumerate([slice(0, half), slice(half, None)]):
        name = f"shard_{m}.{ext}"
        pp.write_shard_file(str(tmp_path / name), gw[sl], c[sl], 64, binary)
        files.append((name, int(len(c[sl]))))
    pp.write_checkpoint_manifest(str(tmp_path), 4, 64, 0.0, files)
    ck = pp.read_checkpoint(str(tmp_path))
    assert ck["layer"] == 4
    assert (ck["words"] == gw).all() and (ck["coeffs"].view(np.uint64) == gc).all()
    json.load(open(tmp_path / "manifest.json"))  # valid JSON


def test_read_checkpoint_errors(pp, tmp_path):
    with pytest.raises(ValueError):
        pp.read_checkpoint(str(tmp_path))  # no manifest
    (tmp_path / "manifest.json").write_text('{"schema": 1, "layer": 2, "qubits": 8, "files": []}\n')
    with pytest.raises(ValueError):
        pp.read_checkpoint(str(tmp_path))  # no shards
    (tmp_path / "manifest.json").write_text('{"layer": 2, "qubits": 8, "files": [{"path": "shard_0.ppb"}]}\n')
    (tmp_path / "shard_0.ppb").write_bytes(b"PPB1" + b"\x00" * 4)
    with pytest.raises(ValueError):
        pp.read_checkpoint(str(tmp_path))  # truncated binary shard
