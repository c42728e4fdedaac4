"""Oracle-backed shard for testing the sharded orchestration on CPU.
TEST INFRASTRUCTURE ONLY: plays the role GpuShard plays on a GPU box, with the
C restatement (oracle/pp_oracle.c) as the local engine, so the protocol of
paper_2506_13241_b200/sharded.py (ownership, eviction, exchange, ingest,
global truncation) is checked against a single-engine oracle run."""
import numpy as np

import oracle as O
from paper_2506_13241_b200 import _pauliprop as _impl
from paper_2506_13241_b200.sharded import SHARD_SEED


class OracleShard:
    def __init__(self, n, epsilon0=0.0):
        self.n = n
        self.eng = O.OracleEngine(n, epsilon0, cadence=1)  # never truncates by itself

    def owner(self, words, world):
        return _impl.shard_owner(np.ascontiguousarray(words, np.uint64).reshape(-1, 4), self.n, SHARD_SEED, world)

    def set_initial(self, words, coeffs):
        self.eng.set_initial(np.ascontiguousarray(words, np.uint64).reshape(-1, 4), np.asarray(coeffs, np.float64))

    def apply_gates(self, gates):
        for g in gates:
            self.eng.apply_gate(np.asarray(g.generator.words, np.uint64), g.cos_theta, g.sin_theta)

    def local_stats(self):
        w, c = self.eng.export()
        nonfinite = bool(np.any(~np.isfinite(c)))
        a = np.abs(c[np.isfinite(c)])
        return (float(a.max()) if a.size else 0.0), nonfinite, int(c.size)

    def truncate_threshold(self, T):
        return self.eng.truncate_threshold(T)

    def record_words(self):
        return 5

    def evict(self, world, rank):
        w, c = self.eng.export()
        own = self.owner(w, world)
        keep = own == rank
        send_order = np.argsort(own[~keep], kind="stable")
        ew, ec = w[~keep][send_order], c[~keep][send_order]
        counts = np.bincount(own[~keep], minlength=world).astype(np.uint64)
        self.eng.set_initial(w[keep], c[keep])
        rec = np.zeros((ew.shape[0], 5), np.uint64)
        rec[:, :4] = ew
        rec[:, 4] = ec.view(np.uint64)
        return rec, counts

    def ingest(self, rec):
        rec = np.asarray(rec, np.uint64).reshape(-1, 5)
        w, c = self.eng.export()
        self.eng.set_initial(np.concatenate([w, rec[:, :4]]), np.concatenate([c, rec[:, 4].copy().view(np.float64)]))

    def term_count(self):
        return self.eng.term_count()

    def expectation(self):
        return self.eng.expectation()

    def export(self):
        return self.eng.export()

    def histogram_counts(self, bins, epsilon0, gmax):
        return self.eng.density_histogram(bins, epsilon0, gmax)
