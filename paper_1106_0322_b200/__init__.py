"""B200-native SMC sparsity-path sampler (drop-in for `spa.smc.run_sampler`).

Lee, Caron, Doucet & Holmes, arXiv:1106.0322.  Host orchestration in
Python/PyTorch; all particle arithmetic in libspa_b200.so (hand-written
sm_100a kernels behind the C ABI declared in include/spa_b200.h).
"""

__version__ = "0.1.0+b200"

from .data import Dataset, SimSpec, named_spec, simulate_dataset  # noqa: F401
from .model import GtPrior  # noqa: F401
from . import summary  # noqa: F401
from .smc import (  # noqa: F401
    DegeneracyError,
    ParticleSystem,
    Schedule,
    SmcConfig,
    SmcOutput,
    StepRecord,
    ess,
    fixed_b_mcmc,
    init_particles,
    load_run,
    make_schedule,
    marginal_summaries,
    reweight,
    run_sampler,
    save_run,
    smc_step,
    systematic_resample,
    systematic_resample_indices,
)
