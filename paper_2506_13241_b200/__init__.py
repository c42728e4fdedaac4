"""B200-native Heisenberg-picture Pauli propagation (drop-in for pauliprop).

Same Python surface as the reference package ``pauliprop``
(python/pauliprop/__init__.py:24-72): ``simulate``, ``PauliString``,
``Gate``, ``Circuit``, ``build_kicked_ising``, ``heavy_hex_127`` ... with the
per-gate branch/merge/truncate and the <0|O|0> readout running as sm_100a
CUDA kernels behind the C-ABI in ``include/pauliprop_gpu.h``.

There is no CPU fallback: importing without the built extension raises, and
creating an engine without a CUDA device raises.
"""
from __future__ import annotations

import os

_HERE = os.path.dirname(os.path.abspath(__file__))


def _nccl_library():
    """The libnccl.so.2 PyTorch links (the nvidia-nccl wheel), so the sharded
    engine's run-time NCCL and a later ``import torch`` share one library."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(base, "nccl", "lib", "libnccl.so.2")
        if os.path.exists(cand):
            return cand
    return None


if "PP_NCCL_LIBRARY" not in os.environ:
    _lib = _nccl_library()
    if _lib:
        os.environ["PP_NCCL_LIBRARY"] = _lib

try:
    from . import _pauliprop as _impl
except ImportError as exc:  # pragma: no cover - exercised only when unbuilt
    raise ImportError(
        "paper_2506_13241_b200: native extension not built "
        "(run `python -m paper_2506_13241_b200.build` or __graft_entry__.build())"
    ) from exc

Circuit = _impl.Circuit
Engine = _impl.Engine
NativeShardedEngine = _impl.NativeShardedEngine
ShardHub = _impl.ShardHub
nccl_unique_id = _impl.nccl_unique_id
Gate = _impl.Gate
Geometry = _impl.Geometry
NumericalError = _impl.NumericalError
PartitionSpec = _impl.PartitionSpec
PauliString = _impl.PauliString
ResourceLimitError = _impl.ResourceLimitError
bfs_ball = _impl.bfs_ball
dump_operator = _impl.dump_operator
histogram_from_counts = _impl.histogram_from_counts
load_dump = _impl.load_dump
read_checkpoint = _impl.read_checkpoint
write_checkpoint_manifest = _impl.write_checkpoint_manifest
write_shard_file = _impl.write_shard_file
build_kicked_ising = _impl.build_kicked_ising
commutes = _impl.commutes
destination_set = _impl.destination_set
heavy_hex_127 = _impl.heavy_hex_127
load_geometry = _impl.load_geometry
load_geometry_file = _impl.load_geometry_file
owner = _impl.owner
parse_circuit = _impl.parse_circuit
parse_pauli_label = _impl.parse_pauli_label
pauli_weight = _impl.pauli_weight
phase_exponent = _impl.phase_exponent
simulate = _impl.simulate
state_vector_expectation = _impl.state_vector_expectation
transfer_totals = _impl.transfer_totals
string_product = _impl.string_product
uniformity_ratio = _impl.uniformity_ratio

NATIVE_LIBS = (
    os.path.join(_HERE, "libppgpu.so"),
    _impl.__file__,
)

__all__ = [
    "Circuit", "Engine", "Gate", "Geometry", "NumericalError", "PartitionSpec",
    "PauliString", "ResourceLimitError", "bfs_ball", "build_kicked_ising",
    "commutes", "destination_set", "dump_operator", "histogram_from_counts", "load_dump", "read_checkpoint",
    "write_checkpoint_manifest", "write_shard_file", "heavy_hex_127", "load_geometry", "load_geometry_file", "owner",
    "parse_circuit", "parse_pauli_label", "pauli_weight", "phase_exponent",
    "simulate", "state_vector_expectation", "string_product", "uniformity_ratio",
]
