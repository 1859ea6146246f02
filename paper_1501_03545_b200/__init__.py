"""B200-native random hyperbolic graph generator.

A drop-in for the generator path of hrgen (arxiv 1501.03545, "Generating
random hyperbolic graphs in subquadratic time"): the same public names for
parameters, sampling, generation, the result Graph and errors, backed by
hand-written sm_100a CUDA behind the C ABI in include/hrgen_b200.h.  There is
no CPU fallback: without libhrgen_b200.so or a CUDA device every generating
call raises NativeLibraryError.
"""

from ._lib import TRIG_CR, TRIG_LIBM
from .engine import Engine, Shard, get_engine
from .errors import (
    InfeasibleParametersError,
    InsufficientDataError,
    NativeLibraryError,
    OutOfBoundsError,
    ParameterDomainError,
)
from .generator import (
    DEFAULT_GENERATOR_CAPACITY,
    GenerationStats,
    GeneratorParams,
    VertexCoordinates,
    add_long_range_edges,
    edges_from_coordinates,
    generate,
    generate_brute_force,
    generate_with_coordinates,
    generate_with_stats,
    radial_inverse_cdf,
    sample_points,
)
from .geometry import (
    TWO_PI,
    ModelParams,
    alpha_from_gamma,
    expected_avg_degree,
    model_constants,
    target_radius,
    to_native_radius,
    to_poincare_radius,
)
from .graph import Graph

__version__ = "0.1.0"

__all__ = [
    "DEFAULT_GENERATOR_CAPACITY", "Engine", "GenerationStats", "GeneratorParams", "Graph",
    "InfeasibleParametersError", "InsufficientDataError", "ModelParams", "NativeLibraryError",
    "OutOfBoundsError", "ParameterDomainError", "Shard", "TRIG_CR", "TRIG_LIBM", "TWO_PI",
    "VertexCoordinates",
    "add_long_range_edges", "alpha_from_gamma", "edges_from_coordinates", "expected_avg_degree",
    "generate", "generate_brute_force", "generate_with_coordinates", "generate_with_stats",
    "get_engine", "model_constants",
    "radial_inverse_cdf", "sample_points", "target_radius", "to_native_radius",
    "to_poincare_radius",
]
