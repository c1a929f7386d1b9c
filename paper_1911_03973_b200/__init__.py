"""paper_1911_03973_b200 -- B200-native element-based P1 finite-element solver path.

Drop-in for the hot path of the reference package ``ebsolve`` (arXiv 1911.03973,
/root/reference/pkg/src/ebsolve/__init__.py:53-92): the same entry-point names
for mesh input, batched K_e/M_e assembly, residual, Dirichlet handling and the
Richardson solver, plus the north-star additions (3D Kuhn tetrahedra, diagonal
extraction, damped Jacobi, CG, Jacobi-PCG, element-slab multi-GPU partition).
Arrays are torch tensors on the CUDA device; the compute is libebs.so
(hand-written sm_100a CUDA behind the C-ABI in include/ebs.h).  There is no CPU
fallback.
"""

from .cli import ExperimentConfig, ExperimentReport, run_experiment
from .elements import (ElementBatch, build_element_batch, combine_system, local_load_batch,
                       local_mass_batch, local_stiffness_batch)
from .mesh import (MAX_LEVEL, IndexArrays, Mesh, boundary_nodes, build_grid_mesh,
                   build_index_arrays, build_unit_cube_mesh, build_unit_square_mesh,
                   export_mesh, face_z0_nodes, jitter_interior, permute_nodes, signed_areas,
                   uniform_refine)
from .operators import (DirichletData, apply_initial_guess, assemble_rhs, constant_dirichlet,
                        diagonal, mask_dirichlet, matvec, residual, residual_many)
from .solvers import (ChebyshevCycle, ConvergenceHistory, SpectralBounds, cg, chebyshev2,
                      chebyshev3, chebyshev_roots, chebyshev_scaling_factor, jacobi, pcg,
                      richardson)
from .reference import dense_interior_eigenvalues, solve_reference
from .sparse import assemble_sparse
from .spectrum import (mass_gershgorin, model_eigen_bounds, model_eigenvalues_all,
                       operator_bounds, power_iteration_lambda_max)

__all__ = [
    "ExperimentConfig", "ExperimentReport", "run_experiment", "solve_reference",
    "dense_interior_eigenvalues",
    "ChebyshevCycle", "chebyshev2", "chebyshev3", "chebyshev_roots", "chebyshev_scaling_factor",
    "mass_gershgorin", "operator_bounds", "power_iteration_lambda_max", "assemble_sparse",
    "uniform_refine", "export_mesh",
    "ConvergenceHistory", "DirichletData", "ElementBatch", "IndexArrays", "MAX_LEVEL", "Mesh",
    "SpectralBounds", "apply_initial_guess", "assemble_rhs", "boundary_nodes",
    "build_element_batch", "build_grid_mesh", "build_index_arrays", "build_unit_cube_mesh",
    "build_unit_square_mesh", "cg", "combine_system", "constant_dirichlet", "diagonal",
    "face_z0_nodes", "jacobi", "jitter_interior", "local_load_batch", "local_mass_batch",
    "local_stiffness_batch", "mask_dirichlet", "matvec", "model_eigen_bounds",
    "model_eigenvalues_all", "pcg", "permute_nodes", "residual", "residual_many", "richardson", "signed_areas",
]

__version__ = "0.1.0"
