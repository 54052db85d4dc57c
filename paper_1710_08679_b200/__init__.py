"""B200-native drop-in for the tetsolve solve path (arXiv 1710.08679).

The compute lives in ``libtsgpu.so`` (hand-written sm_100a CUDA + C++ host,
C ABI in include/tsgpu.h). This package is a thin ctypes mirror of the
reference interface for tests, benchmarks and Python users.
"""
from .tetsolve import (  # noqa: F401
    ConvergenceError,
    DeviceError,
    EbeOperator,
    Error,
    InnerLoopConfig,
    Material,
    Mesh,
    ParseError,
    CrustModel,
    SolveReport,
    SolverLevels,
    build_crust_model,
    build_solver_levels,
    solve,
    solve_pcge,
    SolverConfig,
    SolverError,
    ValidationError,
    dirichlet_mask,
    generate_box_mesh,
    material_from_wavespeeds,
    read_dirichlet,
    read_mesh,
    read_mesh_binary,
    read_solution,
    write_dirichlet,
    write_mesh,
    write_mesh_binary,
    write_solution,
)
