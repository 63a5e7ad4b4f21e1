"""Batch supply for the engine (reference: data.py:1-149).

``gen_teacher_dataset`` / ``batch_iter`` / ``epoch_stream`` restate the
reference's deterministic supply (same SeededRng streams, drop_last,
per-(seed, epoch) permutation), so reference-style MLP runs can be fed
unchanged. ``synthetic_batches`` is the BASELINE workloads' input: x ~ N(0,1)
in (C,H,W) order from SeededRng(seed).normal, labels floor(uniform * C) from
SeededRng(derive_seed(seed, 1)). ``DeviceBatch`` lets a stream hand the engine
batches that already live in HBM (packed bf16 NHWC), which is how bench.py
measures with inputs resident on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .rng import SeededRng, derive_seed


@dataclass
class Dataset:
    inputs: np.ndarray
    labels: np.ndarray

    def __post_init__(self):
        if self.inputs.shape[0] != self.labels.shape[0]:
            raise ValueError(f"inputs ({self.inputs.shape[0]}) and labels ({self.labels.shape[0]}) disagree on N")

    @property
    def n(self) -> int:
        return self.inputs.shape[0]


@dataclass(frozen=True)
class TeacherSpec:
    dims: tuple
    n: int
    seed: int


def gen_teacher_dataset(spec: TeacherSpec) -> Dataset:
    """Teacher weights first, then inputs, from one stream; labels = argmax (data.py:55-77)."""
    rng = SeededRng(spec.seed)
    ws = [rng.normal(a * b).reshape(a, b) / np.sqrt(a) for a, b in zip(spec.dims[:-1], spec.dims[1:])]
    x = rng.normal(spec.n * spec.dims[0]).reshape(spec.n, spec.dims[0])
    h = x
    for i, w in enumerate(ws):
        h = h @ w
        if i < len(ws) - 1:
            h = np.tanh(h)
    return Dataset(x, np.argmax(h, axis=1).astype(np.int64))


def batch_iter(dataset: Dataset, batch_size: int, shuffle_seed: int, epoch: int):
    """drop_last batches under the (seed, epoch) permutation (data.py:133-141)."""
    if batch_size <= 0 or batch_size > dataset.n:
        raise ValueError(f"batch size must lie in [1, {dataset.n}], got {batch_size}")
    perm = SeededRng(derive_seed(shuffle_seed, epoch)).permutation(dataset.n)
    for i in range(dataset.n // batch_size):
        idx = perm[i * batch_size:(i + 1) * batch_size]
        yield dataset.inputs[idx], dataset.labels[idx]


def epoch_stream(dataset: Dataset, batch_size: int, shuffle_seed: int):
    epoch = 0
    while True:
        yield from batch_iter(dataset, batch_size, shuffle_seed, epoch)
        epoch += 1


def synthetic_batches(n_batches: int, batch: int, in_shape, num_classes: int, seed: int = 0):
    width = int(np.prod(in_shape))
    rx = SeededRng(seed)
    rl = SeededRng(derive_seed(seed, 1))
    out = []
    for _ in range(n_batches):
        x = rx.normal(batch * width).reshape(batch, width)
        lab = np.minimum((rl.uniform(batch) * num_classes).astype(np.int64), num_classes - 1)
        out.append((x, lab))
    return out


@dataclass
class DeviceBatch:
    """A batch already resident on the device: packed NHWC activations (the engine's storage
    dtype) + int64 labels."""

    act: object
    labels: object

    @property
    def shape(self):
        return (int(self.labels.shape[0]),)


def to_device_batches(batches, in_shape, device=None, stream=None, precision: str = "bf16"):
    """Pack host batches once into device-resident DeviceBatch objects."""
    from . import _lib as L
    from .runtime import pack_input, require_cuda, torch_mod

    torch = torch_mod()
    dev = require_cuda(device)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    out = []
    for x, lab in batches:
        act = pack_input(np.asarray(x), tuple(in_shape), dev, st, dtype=L.storage_dtype(precision))
        with torch.cuda.stream(st):
            labd = torch.from_numpy(np.asarray(lab, dtype=np.int64)).to(dev)
        out.append(DeviceBatch(act, labd))
    st.synchronize()
    return out


def device_synthetic_batches(n_batches: int, batch: int, in_shape, num_classes: int, seed: int = 0, device=None,
                             stream=None, precision: str = "bf16"):
    """``to_device_batches(synthetic_batches(...))`` generated on the device (csrc/synth.cu): the
    counter-based stream is evaluated per element straight into packed storage-dtype slots, no host
    arrays and no H2D copies."""
    import ctypes as C

    from . import _lib as L
    from .runtime import ptr, require_cuda, stream_ptr, torch_mod

    torch = torch_mod()
    dev = require_cuda(device)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    c, h, w = (tuple(in_shape) + (1, 1))[:3] if len(in_shape) < 3 else tuple(in_shape)
    cp = (c + 7) // 8 * 8
    lib = L.load()
    dt = L.storage_dtype(precision)
    out = []
    for i in range(n_batches):
        with torch.cuda.stream(st):
            act = torch.empty(batch * h * w * cp, dtype=L.torch_storage(dt), device=dev)
            lab = torch.empty(batch, dtype=torch.int64, device=dev)
        L.check(lib.dsp_synth_batch(seed & ((1 << 64) - 1), i, batch, c, h, w, cp, num_classes, dt,
                                    ptr(act), C.cast(ptr(lab), C.POINTER(C.c_int64)), stream_ptr(st)))
        out.append(DeviceBatch(act, lab))
    return out


def cycle(pool):
    while True:
        for b in pool:
            yield b
