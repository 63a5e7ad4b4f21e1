"""paper_1909_02625_b200: B200-native Diversely Stale Parameters (DSP) train step.

Drop-in for the reference package ``stalepipe``'s hot path
(/root/reference/pkg/src/stalepipe/__init__.py): the same names for block
partitioning, queue sizing, the train engine and the optimizer, with
``TrainEngine(..., backend="b200")`` running every tensor operation in
hand-written sm_100a CUDA kernels (libdsp_b200.so, C ABI in include/dsp_b200.h).
Importing the package needs neither a GPU nor the library; constructing a
device engine needs both and fails loudly otherwise (no CPU fallback).
"""

__version__ = "0.1.0"

from ._lib import B200Unavailable, DspError
from .blocks import (
    Block,
    LayerSpec,
    Model,
    ShapeError,
    avgpool,
    basic_unit,
    bottleneck,
    build_model,
    conv_bn_relu,
    dense,
    flop_balanced_boundaries,
    init_params,
    maxpool,
    relu,
    resnet50_layers,
    resnet_cifar_bottleneck_layers,
    resnet_cifar_layers,
    suggest_boundaries,
    tanh,
)
from .data import Dataset, TeacherSpec, batch_iter, epoch_stream, gen_teacher_dataset
from .deviation import DeviationRow, DeviceOperators
from .native import NativeEngine
from .optim import LrSchedule, NonFiniteError, OptimizerState, adam_step, apply_update, lr_at, sgd_step, sum_step
from .pipeline import (
    ActivationPacket,
    ConfigError,
    DeadlockError,
    DeviceStraggler,
    GradPacket,
    LogRecord,
    PipelineConfig,
    ProtocolError,
    RuntimeStraggler,
    StalenessProfile,
    TrainEngine,
    TrainLog,
    default_placement,
    default_queue_config,
    staleness_of,
    validate_config,
)
from .rng import SeededRng, derive_seed, mix64

__all__ = [
    "ActivationPacket", "B200Unavailable", "Block", "ConfigError", "DeadlockError", "DspError", "GradPacket",
    "LayerSpec", "LogRecord", "NativeEngine", "LrSchedule", "Model", "NonFiniteError", "OptimizerState", "PipelineConfig",
    "ProtocolError", "RuntimeStraggler", "SeededRng", "ShapeError", "StalenessProfile", "TrainEngine", "TrainLog",
    "adam_step", "apply_update", "avgpool", "basic_unit", "bottleneck", "build_model", "conv_bn_relu", "default_placement",
    "default_queue_config", "dense", "derive_seed", "flop_balanced_boundaries", "init_params", "lr_at", "maxpool",
    "mix64", "relu", "resnet50_layers", "resnet_cifar_bottleneck_layers", "resnet_cifar_layers", "sgd_step",
    "staleness_of", "suggest_boundaries", "sum_step", "tanh", "validate_config",
    "Dataset", "TeacherSpec", "batch_iter", "epoch_stream", "gen_teacher_dataset", "DeviationRow", "DeviceOperators", "DeviceStraggler",
]
