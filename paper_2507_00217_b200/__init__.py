"""B200-native CrossPipe hot path (arXiv 2507.00217): batched pipeline-schedule
evaluation (§3.5 performance model), greedy schedule generation (Alg. 1) and
grid sweeps with NCCL argmin.  The compute is in libcrosspipe.so (sm_100a);
this package is a thin binding.  Importing it loads the library and fails loudly
if it is missing -- there is no CPU fallback.
"""
from . import _lib

_lib.load()

from .api import (  # noqa: E402,F401
    KEY_NONE, KEY_OVER, HostPipeline, Instances, bubble_ratios, build_static, decode_key, exact, exact_bnb, greedy, pack_instances, quantize,
    records_to_device, ring_hint, sweep_shard_rank,
    simulate, sweep_partition, sweep_shard, to_cp_grid, validate_record,
)

__all__ = ["Instances", "simulate", "greedy", "exact", "exact_bnb", "build_static", "bubble_ratios", "sweep_shard", "sweep_shard_rank", "sweep_partition", "quantize", "decode_key",
           "pack_instances", "records_to_device", "ring_hint", "to_cp_grid", "validate_record"]
