"""B200-native TLED thermo-visco-elastodynamic step (arXiv 2009.10400), behind the
reference's ``tve::Engine`` surface.  See DESIGN.md."""
from .engine import (HALO_NCCL, HALO_PEER, CudaError, Engine, InstabilityError, IoError, NcclError,  # noqa: F401
                     ParseError, TveError,
                     ValidationError, build, critical_timestep, lib, load_mesh, nccl_unique_id, plan)
from .problem import (COUPLED, EXP_ISOTROPIC, EXP_ORTHOTROPIC, EXP_TRANSVERSELY_ISOTROPIC, H8,  # noqa: F401
                      MECHANICAL_ONLY, T4, THERMAL_ONLY, Prescribed, Problem, SourceRegion)
