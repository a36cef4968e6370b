"""B200-native TLED thermo-visco-elastodynamic step (arXiv 2009.10400), behind the
reference's ``tve::Engine`` surface.  See DESIGN.md."""
from .engine import (CudaError, Engine, InstabilityError, IoError, NcclError, ParseError, TveError,  # noqa: F401
                     ValidationError, build, critical_timestep, lib, load_mesh, nccl_unique_id, plan)
from .problem import (COUPLED, EXP_ISOTROPIC, EXP_ORTHOTROPIC, EXP_TRANSVERSELY_ISOTROPIC, H8,  # noqa: F401
                      MECHANICAL_ONLY, T4, THERMAL_ONLY, Prescribed, Problem, SourceRegion)
