"""B200-native DDPMA hot path of arXiv 2006.14602 (drop-in for ``ddmesh``'s
PMA/DDPMA solver and mesh-assembly entry points).

Public names follow the reference package (ddmesh/__init__.py:9-44) for the
hot path: grids and decompositions, density monitors, ``SolverConfig``,
``solve``, ``solve_single_domain``, ``SolveResult``, ``residual`` and the
operator-level PMA functions.  All numerics run in libddpma.so (sm_100a
CUDA); see DESIGN.md.
"""

from .errors import (ConfigurationError, DdmeshError, DomainError,
                     InvalidMonitorError, MeshFileError, StiffnessError)
from .grid import (INTERFACE, PHYSICAL, BoxGeometry, CompGrid, Decomposition,
                   Subdomain, build_decomposition, build_grid, grid_geometry,
                   subdomain_geometry)
from .integrate import (FrozenPmaRhs, IntegrationWindow, advance_window, frozen_rhs,
                        make_integrator, rkc_coeffs)
from .monitor import (ArcLengthDensity, MixtureDensity, MonitorField, RingDensity,
                      ShellDensity, TestFunction, UniformDensity, arc_length_monitor,
                      density_monitor, normalize, SampledField,
                      sampled_field_from_csv, sampled_field_from_vtk, seeded_mixture,
                      test_function_registry)
from .schwarz import (PhysicalMesh, SolverConfig, SolveResult, SubdomainState, WindowRecord,
                      alternating_sweep, init_states, parallel_sweep, residual, solve,
                      solve_single_domain)
from .fileio import (read_mesh_vtk, read_scalar_field_vtk, write_field_csv, write_mesh_vtk,
                     write_scalar_field_vtk)
from .pma import (PotentialField, gradient_fd, hessian_det_fd, initial_potential,
                  physical_mesh, pma_rhs, pma_rhs_frozen)
from .metrics import (ErrorReport, QualityReport, SlopeFit, convergence_slope, quality_measure,
                      quasi1d_oracle, relative_errors, restrict_to_grid)

__version__ = "0.1.0"

__all__ = [
    "CompGrid", "Decomposition", "Subdomain", "build_grid", "build_decomposition",
    "grid_geometry", "subdomain_geometry", "BoxGeometry", "PHYSICAL", "INTERFACE",
    "MonitorField", "density_monitor", "UniformDensity", "RingDensity",
    "ShellDensity", "MixtureDensity", "seeded_mixture",
    "TestFunction", "ArcLengthDensity", "arc_length_monitor", "test_function_registry", "normalize",
    "SampledField", "sampled_field_from_csv", "sampled_field_from_vtk",
    "IntegrationWindow", "rkc_coeffs", "advance_window", "make_integrator", "frozen_rhs",
    "FrozenPmaRhs",
    "SolverConfig", "SolveResult", "WindowRecord", "PhysicalMesh", "PotentialField",
    "solve", "solve_single_domain", "residual", "pma_rhs", "pma_rhs_frozen",
    "initial_potential", "gradient_fd", "hessian_det_fd", "physical_mesh",
    "alternating_sweep", "parallel_sweep", "init_states", "SubdomainState",
    "DdmeshError", "ConfigurationError", "DomainError", "InvalidMonitorError",
    "MeshFileError", "StiffnessError",
    "write_mesh_vtk", "write_scalar_field_vtk", "write_field_csv", "read_mesh_vtk",
    "read_scalar_field_vtk",
    "QualityReport", "ErrorReport", "SlopeFit", "quality_measure", "relative_errors",
    "convergence_slope", "quasi1d_oracle", "restrict_to_grid",
]
