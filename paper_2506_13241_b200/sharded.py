"""Sharded propagation: one engine per rank, strings owned by a hash of their
z-plane.

Why the z-plane: an Rx gate (generator X_q) keeps z, so its branch + merge is
rank-local with no exchange; only runs of Clifford ZZ gates and Z/Y-carrying
generators change z.  After such a run every rank evicts the z-groups it no
longer owns and the others ingest them (equal keys combine exactly like
TermMap::add, so results do not depend on the rank count -- the reference's
own contract, test_engine.cpp:211-258).  Global quantities are collectives:
the per-gate max for relative truncation (engine.cpp:321-345) when
epsilon0 > 0, the term count for the budget check (engine.cpp:266-275), and
the <0|O|0> sum (sparse_operator.cpp:89-97).

The orchestration is SPMD and backend-agnostic: each rank drives a local
``backend`` (the GPU engine, ``GpuShard``) through a ``Comm``.  ``TorchComm``
uses torch.distributed (NCCL or gloo); ``ThreadComm`` runs several ranks as
threads of one process.  The exchange is host-staged in this version.
"""
from __future__ import annotations

import os
import threading
from typing import List, Sequence

import numpy as np

SHARD_SEED = 0x243F6A8885A308D3  # fixed: owner() must agree across ranks


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------
class Comm:
    rank: int = 0
    world: int = 1

    def allreduce(self, values: np.ndarray, op: str) -> np.ndarray:  # op: "sum" | "max"
        raise NotImplementedError

    def alltoallv(self, send: List[np.ndarray]) -> List[np.ndarray]:
        raise NotImplementedError

    def allgather(self, obj) -> list:
        raise NotImplementedError


class TorchComm(Comm):
    """torch.distributed: scalars and the host-staged exchange on `group`
    (CPU tensors, a gloo group); with `data_group` (an NCCL group) the string
    exchange stays on the device: one NCCL all-to-all over NVLink between the
    engines' device buffers (device_exchange)."""

    def __init__(self, group=None, data_group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.data_group = data_group
        self.device_exchange = data_group is not None
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def alltoallv_device(self, send, counts):
        """send: flat int64 CUDA tensor grouped by destination, counts: int64
        words per destination.  Returns (recv tensor, recv word counts)."""
        import torch
        dev = send.device
        c = torch.tensor(counts, dtype=torch.int64, device=dev)
        rc = torch.empty_like(c)
        self.dist.all_to_all_single(rc, c, group=self.data_group)
        rcl = rc.tolist()
        recv = torch.empty(int(sum(rcl)), dtype=torch.int64, device=dev)
        self.dist.all_to_all_single(recv, send, output_split_sizes=rcl, input_split_sizes=list(counts),
                                    group=self.data_group)
        torch.cuda.current_stream(dev).synchronize()
        return recv, rcl

    def allreduce(self, values, op):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64).copy())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM if op == "sum" else self.dist.ReduceOp.MAX, group=self.group)
        return t.numpy()

    def alltoallv(self, send):
        import torch
        counts = np.array([a.size for a in send], np.int64)
        recv_counts = torch.zeros(self.world, dtype=torch.int64)
        self.dist.all_to_all_single(recv_counts, torch.from_numpy(counts), group=self.group)
        rc = recv_counts.numpy()
        flat = np.concatenate([np.ascontiguousarray(a, np.uint64).ravel() for a in send]) if send else np.zeros(0, np.uint64)
        out = torch.zeros(int(rc.sum()), dtype=torch.int64)
        self.dist.all_to_all_single(out, torch.from_numpy(flat.view(np.int64)), output_split_sizes=rc.tolist(),
                                    input_split_sizes=counts.tolist(), group=self.group)
        o = out.numpy().view(np.uint64)
        res, pos = [], 0
        for c in rc:
            res.append(o[pos:pos + c])
            pos += c
        return res

    def allgather(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


class _ThreadHub:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world


class ThreadComm(Comm):
    """Ranks as threads of one process (emulates a multi-GPU run on one GPU;
    no kernel ever waits on another rank).  device=True exchanges device
    buffers (the NCCL path's data flow, with device-to-device copies standing
    in for the all-to-all)."""

    def __init__(self, hub: _ThreadHub, rank: int, device: bool = False):
        self.hub = hub
        self.rank = rank
        self.world = hub.world
        self.device_exchange = device

    @staticmethod
    def make(world, device=False):
        hub = _ThreadHub(world)
        return [ThreadComm(hub, r, device) for r in range(world)]

    def alltoallv_device(self, send, counts):
        import torch
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        allv = self._exchange((send, offs))
        parts = [allv[s][0][int(allv[s][1][self.rank]):int(allv[s][1][self.rank + 1])] for s in range(self.world)]
        recv = torch.cat(parts) if parts else send[:0]
        torch.cuda.current_stream(send.device).synchronize()
        self.hub.barrier.wait()  # every rank holds its copy before any source buffer is reused
        return recv, [int(allv[s][1][self.rank + 1] - allv[s][1][self.rank]) for s in range(self.world)]

    def _exchange(self, obj):
        self.hub.slots[self.rank] = obj
        self.hub.barrier.wait()
        everything = list(self.hub.slots)
        self.hub.barrier.wait()
        return everything

    def allreduce(self, values, op):
        allv = self._exchange(np.asarray(values, np.float64))
        return np.sum(allv, axis=0) if op == "sum" else np.max(allv, axis=0)

    def alltoallv(self, send):
        allv = self._exchange(send)
        return [allv[s][self.rank] for s in range(self.world)]

    def allgather(self, obj):
        return self._exchange(obj)


# ---------------------------------------------------------------------------
# the GPU backend
# ---------------------------------------------------------------------------
class _DeviceWords:
    """__cuda_array_interface__ over an engine-owned device buffer (zero copy)."""

    def __init__(self, ptr, words):
        self.__cuda_array_interface__ = {"shape": (words,), "typestr": "<i8", "data": (ptr, False),
                                         "version": 3, "strides": None}

class GpuShard:
    """One rank's local engine: the CUDA engine with external truncation."""

    def __init__(self, n, epsilon0=0.0, cadence="gate", device=0):
        from . import _pauliprop as _impl
        self.impl = _impl
        self.n = n
        self.device = device
        self.engine = _impl.Engine(n, epsilon0, cadence, device=device, external_truncation=True)

    def owner(self, words, world):
        return self.impl.shard_owner(np.ascontiguousarray(words, np.uint64).reshape(-1, 4), self.n, SHARD_SEED, world)

    def set_initial(self, words, coeffs):
        self.engine.set_initial(np.ascontiguousarray(words, np.uint64).reshape(-1, 4), np.asarray(coeffs, np.float64))

    def apply_gates(self, gates):
        self.engine.apply_gates(list(gates))

    def local_stats(self):
        return self.engine.local_stats()

    def truncate_threshold(self, T):
        return self.engine.truncate_threshold(T)

    def evict(self, world, rank):
        rec, counts = self.engine.shard_evict(world, rank, SHARD_SEED)
        return np.ascontiguousarray(rec), counts

    def evict_device(self, world, rank):
        """Records stay on the device: (flat int64 CUDA tensor view of the
        engine's buffer, records per destination)."""
        import torch
        ptr, counts = self.engine.shard_evict_device(world, rank, SHARD_SEED)
        words = int(sum(counts)) * self.engine.record_words()
        if words == 0:
            return torch.zeros(0, dtype=torch.int64, device=f"cuda:{self.device}"), counts
        return torch.as_tensor(_DeviceWords(ptr, words), device=f"cuda:{self.device}"), counts

    def ingest_device(self, recv, nrec):
        if nrec:
            self.engine.shard_ingest_device(recv.data_ptr(), nrec)

    def ingest(self, rec):
        rw = self.engine.record_words()
        self.engine.shard_ingest(np.ascontiguousarray(rec, np.uint64).reshape(-1, rw))

    def record_words(self):
        return self.engine.record_words()

    def term_count(self):
        return self.engine.term_count()

    def expectation(self):
        return self.engine.expectation_zero_state()

    def export(self):
        return self.engine.export()

    def take_counters(self):
        return self.engine.take_counters()

    def histogram_counts(self, bins, epsilon0, gmax):
        h = self.engine.density_histogram(bins, epsilon0, gmax)
        return np.asarray(h["positive_counts"], np.uint64), np.asarray(h["negative_counts"], np.uint64)


def _is_local(gate) -> bool:
    """Generators that never change z (a single X): rank-local branch."""
    w = np.asarray(gate.generator.words, np.uint64)
    codes = []
    for word in w:
        v = int(word)
        for s in range(32):
            c = (v >> (2 * s)) & 3
            if c:
                codes.append(c)
    return len(codes) == 1 and codes[0] == 1


def _is_clifford(gate) -> bool:
    return gate.cos_theta == 0.0 and gate.sin_theta in (1.0, -1.0)


class ShardedEngine:
    """SPMD driver: same results as one engine, strings spread over ranks."""

    def __init__(self, backend, n, comm: Comm, epsilon0=0.0, cadence="gate", max_terms=0):
        self.b = backend
        self.n = n
        self.comm = comm
        self.eps = float(epsilon0)
        self.per_gate = cadence != "layer"
        self.max_terms = int(max_terms)
        self.gmax = 0.0
        self.exchanged_records = 0

    # -- state
    def set_initial(self, words, coeffs):
        words = np.ascontiguousarray(words, np.uint64).reshape(-1, 4)
        coeffs = np.asarray(coeffs, np.float64)
        own = self.b.owner(words, self.comm.world) == self.comm.rank
        self.b.set_initial(words[own], coeffs[own])
        local = np.abs(coeffs[own]) if own.any() else np.zeros(1)
        finite = local[local == local]
        self.gmax = float(self.comm.allreduce(np.array([finite.max() if finite.size else 0.0]), "max")[0])

    # -- collectives
    def _exchange(self):
        if getattr(self.comm, "device_exchange", False) and hasattr(self.b, "evict_device"):
            rw = self.b.record_words()
            send, counts = self.b.evict_device(self.comm.world, self.comm.rank)
            recv, rwords = self.comm.alltoallv_device(send, [int(c) * rw for c in counts])
            self.exchanged_records += int(sum(int(c) for c in counts))
            self.b.ingest_device(recv, int(sum(rwords)) // rw)
            return
        rec, counts = self.b.evict(self.comm.world, self.comm.rank)
        rw = self.b.record_words()
        send, pos = [], 0
        for c in counts:
            send.append(rec[pos:pos + int(c)])
            pos += int(c)
        got = self.comm.alltoallv(send)
        incoming = np.concatenate([g.reshape(-1, rw) for g in got]) if got else np.zeros((0, rw), np.uint64)
        self.exchanged_records += int(sum(int(c) for c in counts))
        if incoming.shape[0]:
            self.b.ingest(incoming)

    def _epilogue(self, truncate: bool, budget: bool):
        gmax, nonfinite, count = self.b.local_stats()
        red = self.comm.allreduce(np.array([gmax, float(nonfinite)]), "max")
        total = int(self.comm.allreduce(np.array([float(count)]), "sum")[0])
        if budget and self.max_terms and total > self.max_terms:
            from . import ResourceLimitError
            raise ResourceLimitError(f"term budget exhausted: |O|={total} exceeds max_terms={self.max_terms}")
        if truncate:
            if red[1] != 0.0:
                from . import NumericalError
                raise NumericalError(f"non-finite coefficient, |O|={total}")
            self.gmax = float(red[0])
            self.b.truncate_threshold(self.eps * self.gmax)  # engine.cpp:345

    # -- gates
    def apply_gates(self, gates: Sequence):
        """Gates in application order (a layer reversed, as run_circuit does)."""
        gates = list(gates)
        coordinated = self.per_gate and (self.eps > 0.0 or self.max_terms)
        i = 0
        while i < len(gates):
            g = gates[i]
            if _is_local(g) and not _is_clifford(g):
                j = i
                while j < len(gates) and _is_local(gates[j]) and not _is_clifford(gates[j]):
                    j += 1
                if coordinated:
                    for k in range(i, j):
                        self.b.apply_gates([gates[k]])
                        self._epilogue(truncate=True, budget=True)
                else:
                    self.b.apply_gates(gates[i:j])
                    if self.max_terms:
                        self._epilogue(truncate=False, budget=True)
                i = j
            elif _is_clifford(g) and not self.max_terms:
                # a fused Clifford run: magnitudes are permuted, so one truncation
                # at the end equals the reference's per-gate truncations
                j = i
                while j < len(gates) and _is_clifford(gates[j]):
                    j += 1
                self.b.apply_gates(gates[i:j])
                self._exchange()
                if self.per_gate:
                    self._epilogue(truncate=True, budget=False)
                i = j
            else:
                self.b.apply_gates([g])
                self._exchange()
                if self.per_gate:
                    self._epilogue(truncate=True, budget=True)
                elif self.max_terms:
                    self._epilogue(truncate=False, budget=True)
                i += 1
        if self.per_gate and not coordinated:
            # epsilon0 == 0: only exact zeros go, the engines already dropped
            # theirs; keep the global max current for the ledger
            self._epilogue(truncate=True, budget=False)

    def truncate_now(self):
        self._epilogue(truncate=True, budget=False)

    # -- readout
    def term_count(self) -> int:
        return int(self.comm.allreduce(np.array([float(self.b.term_count())]), "sum")[0])

    def expectation_zero_state(self) -> float:
        return float(self.comm.allreduce(np.array([self.b.expectation()]), "sum")[0])

    def export(self):
        w, c = self.b.export()
        parts = self.comm.allgather((np.asarray(w), np.asarray(c)))
        words = np.concatenate([p[0].reshape(-1, 4) for p in parts])
        coeffs = np.concatenate([p[1] for p in parts])
        order = np.lexsort((words[:, 0], words[:, 1], words[:, 2], words[:, 3]))
        return words[order], coeffs[order]

    # -- diagnostics and checkpoints
    def density_histogram(self, bins, epsilon0=None):
        """Global density histogram (sparse_operator.cpp:150-197): per-rank
        device counts summed over ranks, normalized once."""
        from . import _pauliprop as _impl
        eps = self.eps if epsilon0 is None else float(epsilon0)
        pos, neg = self.b.histogram_counts(bins, eps, self.gmax)
        tot = self.comm.allreduce(np.concatenate([pos, neg]).astype(np.float64), "sum")  # exact below 2^53
        tot = tot.astype(np.uint64)
        return _impl.histogram_from_counts(bins, eps, tot[:bins].tolist(), tot[bins:].tolist())

    def write_checkpoint(self, directory, layer, binary=False):
        """runner.cpp:52-77 layout: every rank writes its own shard file,
        rank 0 the manifest."""
        from . import _pauliprop as _impl
        os.makedirs(directory, exist_ok=True)
        w, c = self.b.export()
        name = f"shard_{self.comm.rank}.{'ppb' if binary else 'txt'}"
        _impl.write_shard_file(os.path.join(directory, name), np.asarray(w), np.asarray(c), self.n, binary)
        files = self.comm.allgather((name, int(len(c))))
        if self.comm.rank == 0:
            _impl.write_checkpoint_manifest(directory, int(layer), self.n, self.eps, files)
        self.comm.allgather(None)  # the manifest exists once any rank returns

    def load_checkpoint(self, directory):
        """Loads a checkpoint written by any rank count (or by the
        reference); each rank keeps the strings it owns.  Returns the layer."""
        from . import _pauliprop as _impl
        ck = _impl.read_checkpoint(directory)
        if ck["qubits"] != self.n:
            raise ValueError(f"checkpoint has {ck['qubits']} qubits, engine {self.n}")
        self.set_initial(ck["words"], ck["coeffs"])
        return int(ck["layer"])

    def run_circuit(self, circuit, start_layer=0, out_dir="", histogram_bins=0, checkpoint_every=0,
                    binary_checkpoint=False):
        """run_circuit (engine.cpp:394-446) over the sharded operator, with
        the runner's per-layer outputs (runner.cpp:173-183) and resume."""
        rows = []
        L = circuit.num_layers()
        if not 0 <= start_layer <= L:
            raise ValueError(f"start_layer {start_layer} outside [0, {L}]")
        for t in range(start_layer + 1, L + 1):
            layer = circuit.layers[L - t]
            self.apply_gates(list(reversed(layer)))
            if not self.per_gate:
                self.truncate_now()
            rows.append({"t": t, "observable": self.expectation_zero_state(), "term_count": self.term_count(),
                         "global_max": self.gmax})
            if out_dir and histogram_bins > 0 and self.gmax > 0:
                h = self.density_histogram(histogram_bins)
                if self.comm.rank == 0:
                    os.makedirs(out_dir, exist_ok=True)
                    with open(os.path.join(out_dir, f"histogram_t{t}.tsv"), "w") as f:
                        f.write(h["tsv"])
            if out_dir and checkpoint_every > 0 and t % checkpoint_every == 0:
                self.write_checkpoint(os.path.join(out_dir, f"checkpoint_t{t}"), t, binary_checkpoint)
        return rows
