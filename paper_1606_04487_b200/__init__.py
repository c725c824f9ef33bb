"""B200-native data-parallel CNN training hot path of Omnivore (arXiv 1606.04487).

Drop-in for the hot-path API of the reference package ``omnisim`` 0.1.0
(/root/reference/pkg/src/omnisim/__init__.py:21-81): the conv operators, the
momentum-SGD engine and training loop, the TinyCNN problem, the compute-group
plan and the g-group schedule -- computed by hand-written sm_100a kernels in
libomni.so (C-ABI: include/omni.h).  Out of scope:
the convex test problems, the HE-model optimiser inputs, the implicit-momentum
estimator and SE curves, autotune and cli.
"""

from .cluster import (ExecutionPlan, PhaseProfile, fc_saturated, he_predict, he_predict_pipelined,
                      momentum_for_groups, power_of_two_divisors, t_conv)
from .nets import FC, Conv, NetSpec, Pool, ReLU
from .sgd import (DIVERGENCE_FACTOR, LOSS_WINDOW, Hyperparams, LossTrace, SGDState, StopRule,
                  TrainingProblem, batch_stream, child_seed, iterations_to_loss, run_sync,
                  service_stream, sgd_step, smoothed, stale_step)
from .tensors import (ConvSpec, LoweredMatrix, Tensor4, blowup_ratio, conv_direct, conv_lowered,
                      gemm, lift, lower, lower_kernel)
from .simulator import (SimConfig, SimEvent, SimTrace, StalenessStats, estimate_implicit_momentum,
                        measured_he, simulate, staleness_stats)


def __getattr__(name):
    if name in ("optimizer", "async_groups", "groups"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    # problems / engine import torch CUDA state lazily
    if name in ("CNNProblem", "TinyCNNProblem", "make_tiny_cnn", "make_cnn", "Batch"):
        from . import problems

        return getattr(problems, name)
    if name == "GpuNet":
        from .engine import GpuNet

        return GpuNet
    raise AttributeError(name)


__version__ = "0.1.0"
