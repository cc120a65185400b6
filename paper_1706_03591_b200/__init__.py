"""B200-native (sm_100a) compressive / dynamic spectral clustering hot path.

Drop-in mirror of the reference package ``cscluster``'s hot-path API
(/root/reference/pkg/src/cscluster/__init__.py:9-51, filter / CSC / dynamic
entry points and their data types), backed by libcscb200.so (CUDA, C ABI in
include/csc_b200.h). Import works without a GPU; every compute call needs one.
"""
from .graphs import Graph, LaplacianMatrix, graphs_equal, laplacian
from .signals import FeatureMatrix, as_seed_sequence, random_signals
from .filters import (EigencountSearchError, FilterConfig, FilterPoly, MatvecCounter, apply_filter,
                      cheb_coeffs, eigencount, find_lambda_k, jackson_damping, release_resident_orders,
                      warm_interval)
from .kmeans import Assignment, KmeansConfig, kmeans, kmeans_cost
from .csc import CscDiagnostics, csc_assign, csc_features
from .dynamic import (DynamicConfig, DynamicState, SequenceError, StepDiagnostics, dynamic_init,
                      dynamic_step, run_sequence)

__version__ = "0.1.0"

__all__ = [
    "Graph", "LaplacianMatrix", "graphs_equal", "laplacian",
    "FeatureMatrix", "as_seed_sequence", "random_signals",
    "EigencountSearchError", "FilterConfig", "FilterPoly", "MatvecCounter", "apply_filter",
    "cheb_coeffs", "eigencount", "find_lambda_k", "jackson_damping", "warm_interval",
    "Assignment", "KmeansConfig", "kmeans", "kmeans_cost",
    "CscDiagnostics", "csc_assign", "csc_features",
    "DynamicConfig", "DynamicState", "SequenceError", "StepDiagnostics", "dynamic_init", "dynamic_step",
    "run_sequence",
]
