"""B200-native (A, B) formation + LOBPCG for manifold-graph embedding (arXiv 2112.07862).

Drop-in for the hot path of the reference package ``manigraph``: the names
below mirror ``manigraph/__init__.py:23-66`` for the embedding path.  The
arithmetic runs in hand-written sm_100a kernels (``csrc/``) behind the C ABI
``include/manigraph_b200.h``; there is no CPU fallback.
"""

__version__ = "0.1.0"

from .core import (  # noqa: F401
    DiagonalScaling,
    EigenResult,
    Embedding,
    Graph,
    OperatorPair,
    SolverConfig,
    SparseSymMatrix,
    TwoHopSets,
    assemble_operator,
    balance_radii,
    build_operator_pair,
    connected_components,
    degree_balancing,
    embed,
    fiedler_value,
    identity_shift,
    laplacian,
    laplacian_eigenmaps,
    lobpcg_smallest,
    repulsion_weight,
    require_converged,
    smallest_above_null,
    spmm,
    two_hop_laplacian,
    two_hop_sets,
)
from .clustering import kmeans, normalize_rows  # noqa: F401
from .knn import knn_graph  # noqa: F401
from .textio import (  # noqa: F401
    load_edge_list,
    load_embedding_bin,
    load_embedding_csv,
    load_graph_bin,
    save_edge_list,
    save_embedding_bin,
    save_embedding_csv,
    save_graph_bin,
)
from .errors import (  # noqa: F401
    ConvergenceError,
    DisconnectedGraphError,
    InputError,
    ManigraphError,
    ParseError,
)
from ._native import NativeUnavailable  # noqa: F401
