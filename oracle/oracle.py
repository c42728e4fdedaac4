"""ctypes front end for the parity checkers.  TEST INFRASTRUCTURE ONLY.

Two checkers live under oracle/:

* ``OracleEngine`` -- oracle/pp_oracle.c, a plain-C restatement of the
  reference's engine (engine.cpp:207-351, term_map.cpp:105-144,
  sparse_operator.cpp:89-97), built by ``__graft_entry__.build()`` into
  oracle/_build/libpporacle.so.
* ``RefEngine`` -- the reference engine itself, compiled from its own sources
  under /root/reference by oracle/build_ref.sh into oracle/_ref/libppref.so
  (the .so travels to the GPU box; /root/reference does not).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module.  The product path never does.

Keys here use the reference's interleaved layout (pauli_string.hpp:28-38):
uint64[N, 4], site i in bits (2i, 2i+1) of word i // 32, I=00 X=01 Y=10 Z=11.
``to_planes``/``from_planes`` convert to and from the x/z bit-planes
(x = lo ^ hi, z = hi; inverse lo = x ^ z, hi = z).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libpporacle.so")
REF_SO = os.path.join(HERE, "_ref", "libppref.so")

_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_dbl = ctypes.c_double
_int = ctypes.c_int

OK, INVALID, NUMERICAL, RESOURCE, OTHER = 0, 2, 3, 4, 5


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


# --------------------------------------------------------------------------
# key layout helpers
# --------------------------------------------------------------------------

_SPREAD = np.array([0], dtype=np.uint64)


def _spread32(v: np.ndarray) -> np.ndarray:
    """Spread the low 32 bits of each uint64 to the even bit positions."""
    v = v.astype(np.uint64) & np.uint64(0xFFFFFFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x0000FFFF0000FFFF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF00FF00FF)
    v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F0F0F0F0F)
    v = (v | (v << np.uint64(2))) & np.uint64(0x3333333333333333)
    v = (v | (v << np.uint64(1))) & np.uint64(0x5555555555555555)
    return v


def _compact32(v: np.ndarray) -> np.ndarray:
    """Inverse of _spread32: gather the even bits into the low 32 bits."""
    v = v.astype(np.uint64) & np.uint64(0x5555555555555555)
    v = (v | (v >> np.uint64(1))) & np.uint64(0x3333333333333333)
    v = (v | (v >> np.uint64(2))) & np.uint64(0x0F0F0F0F0F0F0F0F)
    v = (v | (v >> np.uint64(4))) & np.uint64(0x00FF00FF00FF00FF)
    v = (v | (v >> np.uint64(8))) & np.uint64(0x0000FFFF0000FFFF)
    v = (v | (v >> np.uint64(16))) & np.uint64(0x00000000FFFFFFFF)
    return v


def to_planes(words: np.ndarray):
    """uint64[N,4] interleaved -> (x uint64[N,2], z uint64[N,2])."""
    words = np.ascontiguousarray(words, dtype=np.uint64).reshape(-1, 4)
    n = words.shape[0]
    x = np.zeros((n, 2), np.uint64)
    z = np.zeros((n, 2), np.uint64)
    for pw in range(2):  # plane word: sites 64*pw .. 64*pw+63
        lo = np.zeros(n, np.uint64)
        hi = np.zeros(n, np.uint64)
        for half in range(2):  # interleaved word 2*pw+half holds 32 sites
            w = words[:, 2 * pw + half]
            lo |= _compact32(w) << np.uint64(32 * half)
            hi |= _compact32(w >> np.uint64(1)) << np.uint64(32 * half)
        x[:, pw] = lo ^ hi
        z[:, pw] = hi
    return x, z


def from_planes(x: np.ndarray, z: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.uint64).reshape(-1, 2)
    z = np.ascontiguousarray(z, dtype=np.uint64).reshape(-1, 2)
    n = x.shape[0]
    out = np.zeros((n, 4), np.uint64)
    for pw in range(2):
        hi = z[:, pw]
        lo = x[:, pw] ^ z[:, pw]
        for half in range(2):
            sh = np.uint64(32 * half)
            out[:, 2 * pw + half] = _spread32(lo >> sh) | (_spread32(hi >> sh) << np.uint64(1))
    return out


def sort_terms(words: np.ndarray, coeffs: np.ndarray):
    """Canonical order: lexicographic over the 4 interleaved words (w3 most
    significant).  Parity compares sorted sets."""
    words = np.ascontiguousarray(words, dtype=np.uint64).reshape(-1, 4)
    order = np.lexsort((words[:, 0], words[:, 1], words[:, 2], words[:, 3]))
    return words[order], np.asarray(coeffs, np.float64)[order]


def site_word(site: int, code: int) -> np.ndarray:
    w = np.zeros(4, np.uint64)
    w[site // 32] = np.uint64(code) << np.uint64(2 * (site % 32))
    return w


# --------------------------------------------------------------------------
# restatement (oracle/pp_oracle.c)
# --------------------------------------------------------------------------

_olib = None


def _oracle_lib():
    global _olib
    if _olib is None:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(ORACLE_SO)
        L.ppo_create.restype = _vp
        L.ppo_create.argtypes = [_int, _dbl, _int, _u64]
        L.ppo_destroy.argtypes = [_vp]
        L.ppo_set_initial.argtypes = [_vp, _vp, _vp, ctypes.c_size_t]
        L.ppo_apply_gate.argtypes = [_vp, _vp, _dbl, _dbl]
        L.ppo_truncate_now.argtypes = [_vp]
        L.ppo_term_count.restype = _u64
        L.ppo_term_count.argtypes = [_vp]
        L.ppo_global_max.restype = _dbl
        L.ppo_global_max.argtypes = [_vp]
        L.ppo_expectation.restype = _dbl
        L.ppo_expectation.argtypes = [_vp]
        L.ppo_coefficient.restype = _dbl
        L.ppo_coefficient.argtypes = [_vp, _vp]
        L.ppo_export.restype = ctypes.c_int64
        L.ppo_export.argtypes = [_vp, _vp, _vp, _u64]
        L.ppo_take_counters.argtypes = [_vp, _vp]
        L.ppo_angle.argtypes = [_dbl, _int, _vp, _vp, _vp]
        L.ppo_phase_exponent.argtypes = [_vp, _vp, _int]
        L.ppo_truncate_threshold.restype = _u64
        L.ppo_truncate_threshold.argtypes = [_vp, _dbl]
        L.ppo_density_histogram.argtypes = [_vp, _int, _dbl, _dbl, _vp, _vp]
        _olib = L
    return _olib


def oracle_angle(value: float, pi_units: bool):
    L = _oracle_lib()
    c, s, r = _dbl(), _dbl(), _dbl()
    L.ppo_angle(value, int(pi_units), ctypes.byref(c), ctypes.byref(s), ctypes.byref(r))
    return c.value, s.value, r.value


def oracle_phase_exponent(a, b, n):
    a = np.ascontiguousarray(a, np.uint64)
    b = np.ascontiguousarray(b, np.uint64)
    return _oracle_lib().ppo_phase_exponent(a.ctypes.data, b.ctypes.data, n)


class OracleEngine:
    """Single-worker restatement of pauliprop::Engine (engine.hpp:131-200)."""

    def __init__(self, n, epsilon0=0.0, cadence=0, max_terms=0):
        self.L = _oracle_lib()
        self.n = n
        self.cadence = cadence
        self.h = self.L.ppo_create(n, float(epsilon0), int(cadence), int(max_terms))
        if not self.h:
            raise OracleError(INVALID, "bad config")

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ppo_destroy(self.h)
            self.h = None

    def set_initial(self, words, coeffs):
        w = np.ascontiguousarray(words, np.uint64).reshape(-1, 4)
        c = np.ascontiguousarray(coeffs, np.float64)
        self._check(self.L.ppo_set_initial(self.h, w.ctypes.data, c.ctypes.data, len(c)))

    def apply_gate(self, gen_words, cos_t, sin_t):
        g = np.ascontiguousarray(gen_words, np.uint64)
        self._check(self.L.ppo_apply_gate(self.h, g.ctypes.data, float(cos_t), float(sin_t)))

    def truncate_now(self):
        self._check(self.L.ppo_truncate_now(self.h))

    def truncate_threshold(self, threshold):
        return int(self.L.ppo_truncate_threshold(self.h, float(threshold)))

    def _check(self, rc):
        if rc:
            raise OracleError(rc)

    def term_count(self):
        return int(self.L.ppo_term_count(self.h))

    def global_max(self):
        return self.L.ppo_global_max(self.h)

    def expectation(self):
        return self.L.ppo_expectation(self.h)

    def coefficient(self, words):
        w = np.ascontiguousarray(words, np.uint64)
        return self.L.ppo_coefficient(self.h, w.ctypes.data)

    def take_counters(self):
        out = np.zeros(4, np.uint64)
        self.L.ppo_take_counters(self.h, out.ctypes.data)
        return {"removed": int(out[0]), "records_sent": int(out[1]), "gates": int(out[2]),
                "batches_sent": int(out[3])}

    def export(self):
        n = self.term_count()
        w = np.zeros((max(n, 1), 4), np.uint64)
        c = np.zeros(max(n, 1))
        k = self.L.ppo_export(self.h, w.ctypes.data, c.ctypes.data, n)
        return sort_terms(w[:k], c[:k])

    def density_histogram(self, bins, epsilon0, gmax=None):
        """Exact per-bin counts (positive, negative) of density_histogram
        (sparse_operator.cpp:150-197) with x = c / gmax."""
        g = self.global_max() if gmax is None else gmax
        pos = np.zeros(bins, np.uint64)
        neg = np.zeros(bins, np.uint64)
        self._check(self.L.ppo_density_histogram(self.h, bins, g, epsilon0, pos.ctypes.data, neg.ctypes.data))
        return pos, neg

    def run_layers(self, gates, layers):
        """run_circuit semantics (engine.cpp:394-446) for a circuit of
        identical layers.  gates: list of (words[4], cos, sin) in circuit
        (forward) order.  Returns one ledger-like dict per layer."""
        rows = []
        for t in range(1, layers + 1):
            for g in reversed(gates):
                self.apply_gate(*g)
            if self.cadence == 1:
                self.truncate_now()
            cnt = self.take_counters()
            rows.append({"t": t, "observable": self.expectation(),
                         "term_count": self.term_count(),
                         "global_max": self.global_max(),
                         "removed": cnt["removed"],
                         "batches_sent": cnt["batches_sent"],
                         "records_sent": cnt["records_sent"]})
        return rows


# --------------------------------------------------------------------------
# the reference itself (oracle/_ref)
# --------------------------------------------------------------------------

_rlib = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _ref_lib():
    global _rlib
    if _rlib is None:
        L = ctypes.CDLL(REF_SO)
        L.ppref_last_error.restype = ctypes.c_char_p
        L.ppref_create.restype = _vp
        L.ppref_create.argtypes = [_int, ctypes.c_uint32, _int, _dbl, _int, _u64]
        L.ppref_destroy.argtypes = [_vp]
        L.ppref_set_initial.argtypes = [_vp, _vp, _vp, ctypes.c_size_t]
        L.ppref_apply_gate.argtypes = [_vp, _vp, _dbl, _int]
        L.ppref_truncate_now.argtypes = [_vp]
        L.ppref_run_circuit.argtypes = [_vp, _int, _vp, _vp, _vp, _vp, _int, _vp]
        L.ppref_time_circuit.argtypes = [_vp, _int, _vp, _vp, _vp, _vp, _int, _vp, _vp]
        L.ppref_term_count.restype = _u64
        L.ppref_term_count.argtypes = [_vp]
        L.ppref_shard_sizes.restype = _int
        L.ppref_shard_sizes.argtypes = [_vp, _vp, _int]
        L.ppref_global_max.restype = _dbl
        L.ppref_global_max.argtypes = [_vp]
        L.ppref_expectation.restype = _dbl
        L.ppref_expectation.argtypes = [_vp]
        L.ppref_export.restype = ctypes.c_int64
        L.ppref_export.argtypes = [_vp, _vp, _vp, _u64]
        L.ppref_coefficient.restype = _dbl
        L.ppref_coefficient.argtypes = [_vp, _vp]
        L.ppref_parse_label.argtypes = [ctypes.c_char_p, _int, _vp]
        L.ppref_phase_exponent.argtypes = [_vp, _vp, _int]
        L.ppref_angle.argtypes = [_dbl, _int, _vp, _vp, _vp]
        L.ppref_heavy_hex.argtypes = [_vp, _vp, _int]
        L.ppref_kicked_layer.argtypes = [ctypes.c_char_p, _vp, _vp, _int]
        L.ppref_histogram_tsv.argtypes = [_vp, _int, _dbl, ctypes.c_char_p, _u64]
        L.ppref_histogram_tsv.restype = ctypes.c_int64
        L.ppref_dump.argtypes = [_vp, ctypes.c_char_p, _u64]
        L.ppref_dump.restype = ctypes.c_int64
        L.ppref_load_dump.argtypes = [ctypes.c_char_p, _int, _vp, _vp, _u64]
        L.ppref_load_dump.restype = ctypes.c_int64
        _rlib = L
    return _rlib


def ref_angle(value: float, pi_units: bool):
    L = _ref_lib()
    c, s, r = _dbl(), _dbl(), _dbl()
    L.ppref_angle(value, int(pi_units), ctypes.byref(c), ctypes.byref(s), ctypes.byref(r))
    return c.value, s.value, r.value


def ref_parse_label(text: str, n: int) -> np.ndarray:
    w = np.zeros(4, np.uint64)
    rc = _ref_lib().ppref_parse_label(text.encode(), n, w.ctypes.data)
    if rc:
        raise OracleError(rc, _ref_lib().ppref_last_error().decode())
    return w


def ref_heavy_hex():
    """(edges [(i, j)], colors [c]) of the reference's bundled map."""
    e = np.zeros(400, np.int32)
    c = np.zeros(200, np.int32)
    k = _ref_lib().ppref_heavy_hex(e.ctypes.data, c.ctypes.data, 200)
    return [(int(e[2 * i]), int(e[2 * i + 1])) for i in range(k)], [int(v) for v in c[:k]]


def ref_kicked_layer(geometry_text: str):
    """Generator words of kicked_ising_layer (models.cpp:149-171), forward order."""
    w = np.zeros(4 * 2048, np.uint64)
    z = np.zeros(2048, np.int32)
    k = _ref_lib().ppref_kicked_layer(geometry_text.encode(), w.ctypes.data, z.ctypes.data, 2048)
    if k < 0:
        raise OracleError(INVALID, _ref_lib().ppref_last_error().decode())
    return w[: 4 * k].reshape(k, 4).copy(), z[:k].astype(bool)


class RefEngine:
    """The reference pauliprop::Engine (oracle/_ref)."""

    def __init__(self, n, epsilon0=0.0, cadence=0, max_terms=0, workers=1, threads=1):
        self.L = _ref_lib()
        self.n = n
        self.h = self.L.ppref_create(n, workers, threads, float(epsilon0), int(cadence), int(max_terms))
        if not self.h:
            raise OracleError(INVALID, self.L.ppref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ppref_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.L.ppref_last_error().decode())

    def set_initial(self, words, coeffs):
        w = np.ascontiguousarray(words, np.uint64).reshape(-1, 4)
        c = np.ascontiguousarray(coeffs, np.float64)
        self._check(self.L.ppref_set_initial(self.h, w.ctypes.data, c.ctypes.data, len(c)))

    def apply_gate(self, gen_words, theta, pi_units):
        g = np.ascontiguousarray(gen_words, np.uint64)
        self._check(self.L.ppref_apply_gate(self.h, g.ctypes.data, float(theta), int(pi_units)))

    def truncate_now(self):
        self._check(self.L.ppref_truncate_now(self.h))

    @staticmethod
    def _flatten(gates):
        words = np.ascontiguousarray(np.stack([np.asarray(g[0], np.uint64) for g in gates]))
        theta = np.array([float(g[1]) for g in gates], np.float64)
        pi = np.array([int(g[2]) for g in gates], np.int32)
        return words, theta, pi

    def run_circuit(self, gates, layers=1):
        """gates: [(words[4], theta, pi_units)] forward order, one layer,
        repeated `layers` times.  Returns ledger rows (engine.hpp:70-79)."""
        words, theta, pi = self._flatten(gates)
        rows = []
        for _ in range(layers):
            out = np.zeros(8)
            sizes = np.array([len(gates)], np.int64)
            self._check(self.L.ppref_run_circuit(self.h, self.n, words.ctypes.data, theta.ctypes.data,
                                                 pi.ctypes.data, sizes.ctypes.data, 1, out.ctypes.data))
            rows.append({"observable": out[1], "term_count": int(out[2]), "global_max": out[3],
                         "removed": int(out[4]), "wall_ms_per_gate": out[5],
                         "batches_sent": int(out[6]), "records_sent": int(out[7])})
        for t, r in enumerate(rows, 1):
            r["t"] = t
        return rows

    def time_circuit(self, gates, layers=1):
        words, theta, pi = self._flatten(gates)
        sizes = np.array([len(gates)] * layers, np.int64)
        words = np.ascontiguousarray(np.tile(words, (layers, 1)))
        theta = np.tile(theta, layers)
        pi = np.tile(pi, layers)
        sec, sg = _dbl(), _dbl()
        self._check(self.L.ppref_time_circuit(self.h, self.n, words.ctypes.data, theta.ctypes.data,
                                              pi.ctypes.data, sizes.ctypes.data, layers,
                                              ctypes.byref(sec), ctypes.byref(sg)))
        return sec.value, sg.value

    def term_count(self):
        return int(self.L.ppref_term_count(self.h))

    def shard_sizes(self):
        out = np.zeros(4096, np.uint64)
        k = self.L.ppref_shard_sizes(self.h, out.ctypes.data, 4096)
        return [int(v) for v in out[:k]]

    def global_max(self):
        return self.L.ppref_global_max(self.h)

    def expectation(self):
        return self.L.ppref_expectation(self.h)

    def coefficient(self, words):
        w = np.ascontiguousarray(words, np.uint64)
        return self.L.ppref_coefficient(self.h, w.ctypes.data)

    def _text(self, fn, *args):
        cap = 1 << 16
        while True:
            buf = ctypes.create_string_buffer(cap)
            r = fn(self.h, *args, buf, cap)
            if r == -1:
                raise OracleError(2, self.L.ppref_last_error().decode())
            if r >= 0:
                return buf.value.decode()
            cap = -r

    def histogram_tsv(self, bins, epsilon0):
        """The reference's density_histogram(...).to_tsv() for this engine."""
        return self._text(self.L.ppref_histogram_tsv, bins, epsilon0)

    def dump(self):
        """Concatenated SparseOperator::dump of all shards."""
        return self._text(self.L.ppref_dump)

    def export(self):
        n = self.term_count()
        w = np.zeros((max(n, 1), 4), np.uint64)
        c = np.zeros(max(n, 1))
        k = self.L.ppref_export(self.h, w.ctypes.data, c.ctypes.data, n)
        return sort_terms(w[:k], c[:k])


def ref_load_dump(text: str, n: int):
    """SparseOperator::load_dump of the reference (sorted words, coeffs)."""
    L = _ref_lib()
    cap = max(1, text.count("\n") + 1)
    w = np.zeros((cap, 4), np.uint64)
    c = np.zeros(cap)
    k = L.ppref_load_dump(text.encode(), n, w.ctypes.data, c.ctypes.data, cap)
    if k < 0:
        raise OracleError(2, L.ppref_last_error().decode())
    return sort_terms(w[:k], c[:k])
