"""paper_1505_00581_b200 -- exact space-time hypergraph matching for action
detection (Lombardi et al., arXiv 1505.00581) on B200 (sm_100a).

The product is libhgm.so (include/hgm.h); `hgm` is its thin Python binding and
`dist` shards offsets across GPUs (one process per GPU, NCCL for the final
gather).  Nothing here imports the test oracle.
"""
from .hgm import (  # noqa: F401
    DevicePoints,
    HGMError,
    Model,
    Params,
    Scene,
    build_model_graph,
    build_scene_index,
    detect_actions,
    get_stats,
    match_model_at_offsets,
    set_profiling,
    version,
)
