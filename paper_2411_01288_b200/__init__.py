"""paper_2411_01288_b200 -- B200-native HEXA-MoE expert-specific MoE-layer hot path.

Drop-in for the reference ``moekit`` operator API (routing / es_ops /
moe_layer, /root/reference/proj/core/include/moekit/) with every kernel a
hand-written sm_100a CUDA kernel behind the C ABI in include/hexamoe.h.
"""
from ._lib import CacheError, HexaMoeCudaError, ShapeError, lib  # noqa: F401
from .es_ops import ACCUMULATE, WRITE, EsfkResult, OpStats, esfk, esmm, ess, estmm  # noqa: F401
from .moe_layer import (ForwardStash, MoeForwardResult, MoeGrads, MoeLayerParams,  # noqa: F401
                        estimate_activation_memory, layer_workspace, make_desc,
                        make_random_params, moe_backward, moe_forward)
from .routing import (ReIndex, RoutingChoice, build_reindex, build_reindex_all,  # noqa: F401
                      read_routing_csv, routing_from_csv, routing_to_csv,
                      synthesize_routing, write_routing_csv)

__version__ = "0.1.0"
