"""paper_2406_02807_b200 -- B200-native CAPT batched collision query.

Drop-in for the hot path of the reference package ``captree`` (arXiv
2406.02807): build a collision-affording point tree from fp32 points with
r_min/r_max, then answer batched sphere queries -- all on sm_100a CUDA
kernels behind the C-ABI in include/capt_b200.h.
"""

from .cloud import PointCloud
from .dispersion import DispersionStats, dispersion_stats, nn_distances, safe_filter_radius
from .geom import Aabb, Sphere
from .morton import FilterConfig, axis_bits, filter_cloud, reach_filter
from .query import (DEFAULT_LANE_WIDTH, QueryOutcome, SphereBatch, collides, collides_any,
                    collides_batch, collides_many, collides_unchecked, query_bits)
from .trace import (ParseError, QueryTraceRecord, VerificationError, capt_verdicts, query_phase,
                    read_trace, verify_trace, write_trace)
from .tree import (BuildParams, BuildStats, Capt, construct, leaf_index, leaf_index_counted,
                   leaf_indices, load_capt, save_capt)

__version__ = "0.1.0"

__all__ = [
    "Aabb", "Sphere", "PointCloud",
    "FilterConfig", "axis_bits", "filter_cloud", "reach_filter",
    "BuildParams", "BuildStats", "Capt", "construct", "leaf_index", "leaf_index_counted",
    "leaf_indices", "save_capt", "load_capt",
    "SphereBatch", "QueryOutcome", "collides", "collides_unchecked", "collides_batch",
    "collides_any", "collides_many", "query_bits", "DEFAULT_LANE_WIDTH",
    "QueryTraceRecord", "ParseError", "VerificationError", "read_trace", "write_trace",
    "capt_verdicts", "verify_trace", "query_phase",
    "DispersionStats", "dispersion_stats", "nn_distances", "safe_filter_radius",
]
