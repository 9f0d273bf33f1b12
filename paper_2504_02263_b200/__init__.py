"""B200-native disaggregated expert-parallel MoE decode step (MegaScale-Infer,
arXiv 2504.02263): config API compatible with the reference ``moeplan``
package, sm_100a CUDA kernels behind a C ABI (libmsinfer.so), NVLink M2N.

Submodules:
  config    -- MoeModelSpec / WorkloadSpec / SearchLimits / config loader (+ plan)
  pipeline  -- ping-pong timing model (Eq. 4/5, simulator) used as the timing oracle
  ops       -- stateless kernels (router, grouped FFN, combine)
  runtime   -- M2N group, MoEDecodeLayer, PingPongRunner (needs a B200)
"""

from .config import (  # noqa: F401
    Catalog, ConfigBundle, ConfigError, DeploymentPlan, GpuSpec, MoeModelSpec, SearchLimits,
    WorkloadSpec, builtin_catalog, builtin_models, config_from_dict, config_to_dict, load_config,
    load_plan, resolve_model, save_config,
)

__version__ = "0.1.0"
