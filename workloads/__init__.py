"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds ONLY input construction (graphs, adjacency matrices, seeded
random matrices).  It contains none of the permanent method's arithmetic, so
both `oracle/` (test infrastructure) and `paper_1112_6072_b200/` (the product)
may import it without sharing any of the method's code.

Workloads (BASELINE.json "configs"):
  configs[0]  dodecahedron C20                       -> dodecahedron()
  configs[1]  256 random n=24 3-regular (weighted)   -> random_3perm_batch()
  configs[2]  C60 truncated icosahedron              -> truncated_icosahedron()
  configs[3]  spiral fullerenes n in {70,76,80,84}   -> spiral_fullerene()
  configs[4]  n=96 random 3-regular + n=96 fullerene -> random_3perm(), spiral_fullerene()
Paper data: appendix C60 / C100 adjacency tables -> paper_graph().
"""
from .graphs import (  # noqa: F401
    adjacency_matrix,
    dodecahedron,
    icosahedron,
    truncated_icosahedron,
    paper_graph,
    random_3perm,
    random_3perm_batch,
    spiral_fullerene,
    spiral_windup,
    random_fullerene,
    random_sparse01,
    face_cycles,
)
