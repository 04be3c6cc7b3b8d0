"""B200-native (sm_100a) Chameleon hot path: batched Adaptive-Exploration rollout
+ GBT cost-model scoring, and Adaptive-Sampling k-means, behind the reference's
ktune interfaces (see include/ktune_cuda.h).

All compute runs in libktune_cuda.so (hand-written CUDA for sm_100a). There is
no CPU fallback: importing a compute entry point without the built library
raises ImportError.
"""
from .errors import BackendError, ConfigError, CudaError, LogicError, SpaceExhaustedError  # noqa: F401
from .spaces import (DesignSpace, Knob, alexnet_tasks, conv_space, mix64, resnet18_tasks,  # noqa: F401
                     seed_combine, small_space, stream_seed, synthetic_space, vgg16_tasks)

__all__ = ["DesignSpace", "Knob", "ConfigError", "BackendError", "SpaceExhaustedError", "LogicError"]


def __getattr__(name):
    # Lazy: the compute API loads libktune_cuda.so on first use.
    import importlib
    if name.startswith("_") or name in ("context", "cost_model", "exploration", "sampling", "spaces",
                                        "errors", "distributed"):
        raise AttributeError(name)
    for mod in ("context", "cost_model", "exploration", "sampling"):
        m = importlib.import_module(f".{mod}", __name__)
        if hasattr(m, name):
            return getattr(m, name)
    raise AttributeError(name)
