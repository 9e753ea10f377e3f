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
from .integrate import IntegrationWindow, rkc_coeffs
from .monitor import (ArcLengthDensity, MixtureDensity, MonitorField, RingDensity,
                      ShellDensity, TestFunction, UniformDensity, arc_length_monitor,
                      density_monitor, normalize, SampledField,
                      sampled_field_from_csv, sampled_field_from_vtk, seeded_mixture,
                      test_function_registry)
from .schwarz import (PhysicalMesh, SolverConfig, SolveResult, WindowRecord,
                      residual, solve, solve_single_domain)
from .fileio import (read_mesh_vtk, read_scalar_field_vtk, write_field_csv, write_mesh_vtk,
                     write_scalar_field_vtk)
from .pma import pma_rhs
from .metrics import (ErrorReport, QualityReport, quality_measure, relative_errors,
                      restrict_to_grid)

__version__ = "0.1.0"

__all__ = [
    "CompGrid", "Decomposition", "Subdomain", "build_grid", "build_decomposition",
    "grid_geometry", "subdomain_geometry", "BoxGeometry", "PHYSICAL", "INTERFACE",
    "MonitorField", "density_monitor", "UniformDensity", "RingDensity",
    "ShellDensity", "MixtureDensity", "seeded_mixture",
    "TestFunction", "ArcLengthDensity", "arc_length_monitor", "test_function_registry", "normalize",
    "SampledField", "sampled_field_from_csv", "sampled_field_from_vtk",
    "IntegrationWindow", "rkc_coeffs",
    "SolverConfig", "SolveResult", "WindowRecord", "PhysicalMesh",
    "solve", "solve_single_domain", "residual", "pma_rhs",
    "DdmeshError", "ConfigurationError", "DomainError", "InvalidMonitorError",
    "MeshFileError", "StiffnessError",
    "write_mesh_vtk", "write_scalar_field_vtk", "write_field_csv", "read_mesh_vtk",
    "read_scalar_field_vtk",
    "QualityReport", "ErrorReport", "quality_measure", "relative_errors", "restrict_to_grid",
]
