"""paper_2505_06771_b200 — B200-native batched Robotarium step (JaxRobotarium's
accelerator contribution), behind the reference mrsim batch-engine interface.

The hot path is hand-written sm_100a CUDA (csrc/), exported as a C ABI
(include/mrsim_cuda.h, libmrsim_cuda.so); this package is the thin host-side
mirror of the reference's reset_batch / step_batch / ScenarioConfig.
"""
from ._lib import (CudaError, DomainError, InvalidArgument, MrsimError, SimRuntimeError, Unsupported,
                   lib)
from .batch import (TASKS, CudaEnvBatch, FeedforwardWeights, ScenarioConfig, StepOutputs, derive_episode_seed,
                    make_default_config, reset_batch, step_batch)

__all__ = [
    "TASKS", "CudaEnvBatch", "FeedforwardWeights", "ScenarioConfig", "StepOutputs", "make_default_config", "reset_batch",
    "step_batch", "derive_episode_seed", "lib", "MrsimError", "InvalidArgument", "DomainError",
    "SimRuntimeError", "CudaError", "Unsupported",
]
