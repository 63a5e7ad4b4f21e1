"""Run/artifact integration with ``train.backend = b200``.

The reference's front door (/root/reference/pkg/src/stalepipe/runners.py:51-167,
config.py:29-201, cli.py:103-119) drives ``TrainEngine`` from a flat ``key = value``
config and writes a TrainLog JSONL, an epoch summary CSV, the Lemma-1 report of the
deviation rows, the resolved config and run metadata. This module reads the same format
and keys, builds this package's model / pipeline / data objects, trains on the B200
engine and writes the same artifacts, so an existing experiment config runs unchanged
with ``train.backend = b200``.

Beyond the reference's layer grammar (``dense(i,o[,bias])``, ``relu``, ``tanh``) the
layer list accepts the CNN kinds and whole-network macros: ``resnet_cifar(depth[,
classes[, width]])``, ``resnet_cifar_bottleneck(depth[, classes])``, ``resnet50([classes])``;
``model.boundaries = auto`` picks FLOP-balanced cuts for ``pipeline.p``'s K. Data sources:
``teacher`` (the reference's) and ``synthetic`` (the benchmark pool).
"""

from __future__ import annotations

import csv
import json
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import blocks as B
from .data import Dataset, TeacherSpec, epoch_stream, gen_teacher_dataset, synthetic_batches
from .optim import LrSchedule
from .pipeline import RuntimeStraggler, TrainEngine, staleness_of, validate_config
from .rng import derive_seed
from .theory import estimate_constants, lemma1_report

SCHEMA_VERSION = 1


class ConfigParseError(ValueError):
    pass


def parse_config_text(text: str) -> dict:
    """``key = value`` lines, ``#`` comments (config.py:29-42)."""
    out = {}
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        if "=" not in line:
            raise ConfigParseError(f"line {lineno}: expected 'key = value', got {raw!r}")
        key, value = line.split("=", 1)
        if not key.strip():
            raise ConfigParseError(f"line {lineno}: empty key")
        out[key.strip()] = value.strip()
    return out


def load_config_file(path) -> dict:
    return parse_config_text(Path(path).read_text())


def render_config(cfg: dict) -> str:
    return "".join(f"{k} = {cfg[k]}\n" for k in sorted(cfg))


def _parse_bool(value: str, what: str) -> bool:
    v = value.strip().lower()
    if v in ("true", "1", "yes"):
        return True
    if v in ("false", "0", "no"):
        return False
    raise ConfigParseError(f"{what}: expected true/false, got {value!r}")


def _split_top(text: str) -> list:
    toks, depth, cur = [], 0, ""
    for ch in text:
        depth += ch == "("
        depth -= ch == ")"
        if ch == "," and depth == 0:
            toks.append(cur)
            cur = ""
        else:
            cur += ch
    if cur.strip():
        toks.append(cur)
    return [t.strip() for t in toks]


def parse_layers(text: str) -> list:
    """The reference's grammar (config.py:54-90) plus CNN network macros."""
    layers = []
    for tok in _split_top(text):
        name, args = tok, []
        if "(" in tok and tok.endswith(")"):
            name = tok[: tok.index("(")].strip()
            args = [a.strip() for a in tok[tok.index("(") + 1: -1].split(",") if a.strip()]
        try:
            if name in ("relu", "tanh") and not args:
                layers.append(B.relu() if name == "relu" else B.tanh())
            elif name == "dense" and len(args) in (2, 3):
                bias = _parse_bool(args[2], f"dense bias in {tok!r}") if len(args) == 3 else True
                layers.append(B.dense(int(args[0]), int(args[1]), bias))
            elif name == "resnet_cifar" and 1 <= len(args) <= 3:
                kw = {"width": int(args[2])} if len(args) == 3 else {}
                layers.extend(B.resnet_cifar_layers(int(args[0]), int(args[1]) if len(args) > 1 else 10, **kw))
            elif name == "resnet_cifar_bottleneck" and 1 <= len(args) <= 2:
                layers.extend(B.resnet_cifar_bottleneck_layers(int(args[0]), int(args[1]) if len(args) > 1 else 100))
            elif name == "resnet50" and len(args) <= 1:
                layers.extend(B.resnet50_layers(int(args[0]) if args else 1000))
            else:
                raise ConfigParseError(f"unknown layer token: {tok!r}")
        except ValueError as exc:
            if isinstance(exc, ConfigParseError):
                raise
            raise ConfigParseError(f"bad layer spec {tok!r}: {exc}") from None
    if not layers:
        raise ConfigParseError("empty layer list")
    return layers


@dataclass
class RunConfig:
    """Typed view over the flat key map (config.py:103-201), building this package's objects."""

    raw: dict = field(default_factory=dict)

    def get(self, key: str, default=None) -> str:
        if key in self.raw:
            return self.raw[key]
        if default is None:
            raise ConfigParseError(f"missing required key: {key}")
        return default

    def get_int(self, key, default=None) -> int:
        raw = self.get(key, None if default is None else str(default))
        try:
            return int(raw)
        except ValueError:
            raise ConfigParseError(f"{key}: expected integer, got {raw!r}") from None

    def get_float(self, key, default=None) -> float:
        raw = self.get(key, None if default is None else repr(default))
        try:
            return float(raw)
        except ValueError:
            raise ConfigParseError(f"{key}: expected number, got {raw!r}") from None

    def get_bool(self, key, default: bool) -> bool:
        return _parse_bool(self.get(key, "true" if default else "false"), key)

    def get_ints(self, key, default=None) -> list:
        raw = self.get(key, default)
        return [] if raw.strip() == "" else [int(v) for v in raw.split(",")]

    def build_pipeline(self):
        return validate_config(self.get_ints("pipeline.p"), self.get_ints("pipeline.m"),
                               warmup=self.get("pipeline.warmup", "faithful_zero_updates"),
                               overlap_recompute=self.get_bool("pipeline.overlap_recompute", True))

    def build_model(self):
        layers = parse_layers(self.get("model.layers"))
        cuts = self.get("model.boundaries", "")
        if cuts.strip() == "auto":
            bounds = B.flop_balanced_boundaries(layers, len(self.get_ints("pipeline.p")))
        else:
            bounds = self.get_ints("model.boundaries", "")
        model = B.build_model(layers, bounds)
        B.init_params(model, self.get_int("model.init_seed", self.get_int("train.seed", 0)))
        return model

    def build_schedule(self) -> LrSchedule:
        steps = self.get_ints("optimizer.lr_decay_steps", "")
        factor = self.get_float("optimizer.lr_decay_factor", 0.1)
        return LrSchedule(base=self.get_float("optimizer.lr", 0.01), decays=tuple((s, factor) for s in steps))

    def build_dataset(self, split: str = "train") -> Dataset:
        source = self.get("data.source", "teacher")
        if source == "teacher":
            dims = tuple(self.get_ints("data.teacher_dims"))
            n_train = self.get_int("data.n_train")
            n_test = self.get_int("data.n_test", 0)
            full = gen_teacher_dataset(TeacherSpec(dims=dims, n=n_train + n_test, seed=self.get_int("data.seed", 0)))
            if split == "train":
                return Dataset(full.inputs[:n_train], full.labels[:n_train])
            return Dataset(full.inputs[n_train:], full.labels[n_train:])
        if source == "synthetic":
            shape = tuple(self.get_ints("data.shape"))
            classes = self.get_int("data.classes")
            bs = self.get_int("data.batch_size", 64)
            n = self.get_int("data.n_train" if split == "train" else "data.n_test", 0)
            seed = self.get_int("data.seed", 0) + (0 if split == "train" else 1)
            pool = synthetic_batches(max(1, n // bs), bs, shape, classes, seed=seed)
            return Dataset(np.concatenate([x for x, _ in pool]), np.concatenate([lab for _, lab in pool]))
        raise ConfigParseError(f"data.source must be 'teacher' or 'synthetic', got {source!r}")


def evaluate(model, dataset: Dataset, batch: int = 512) -> tuple:
    """Full-pass mean loss and accuracy at the model's current parameters (runners.py:51-56),
    forward on the device in chunks of ``batch`` samples."""
    n = dataset.inputs.shape[0]
    loss_sum, correct = 0.0, 0
    for i in range(0, n, batch):
        x, y = dataset.inputs[i:i + batch], dataset.labels[i:i + batch]
        z = model.forward(x).astype(np.float64)
        z = z - z.max(axis=1, keepdims=True)
        logp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
        loss_sum += float(-logp[np.arange(len(y)), y].sum())
        correct += int((np.argmax(z, axis=1) == y).sum())
    return loss_sum / n, correct / n


def run_validate(cfg: RunConfig) -> dict:
    pipe = cfg.build_pipeline()
    prof = staleness_of(pipe)
    return {"k": pipe.k, "p": list(pipe.p), "m": list(pipe.m), "q": list(pipe.q),
            "staleness": list(prof.per_block), "max_staleness": prof.max, "warmup": pipe.warmup}


def run_train(cfg: RunConfig, out_dir) -> dict:
    """Train with ``train.backend = b200`` and write the reference's artifacts (runners.py:59-167)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    backend = cfg.get("train.backend", "b200")
    if backend != "b200":
        raise ConfigParseError(f"train.backend must be 'b200' for this package, got {backend!r}")
    model = cfg.build_model()
    pipe = cfg.build_pipeline()
    train_ds = cfg.build_dataset("train")
    test_ds = cfg.build_dataset("test") if cfg.get_int("data.n_test", 0) else None
    batch_size = cfg.get_int("data.batch_size", 64)
    seed = cfg.get_int("train.seed", 0)
    straggler = None
    if cfg.get_float("train.straggler_prob", 0.0) > 0:
        straggler = RuntimeStraggler(prob=cfg.get_float("train.straggler_prob", 0.0),
                                     delay_s=cfg.get_float("train.straggler_delay_ms", 1.0) / 1e3,
                                     seed=cfg.get_int("train.straggler_seed", seed))
    engine = TrainEngine(model, pipe, epoch_stream(train_ds, batch_size, shuffle_seed=derive_seed(seed, 1)),
                         schedule=cfg.build_schedule(), rule=cfg.get("optimizer.rule", "sgd"),
                         beta=cfg.get_float("optimizer.beta", 0.9), s=cfg.get_float("optimizer.s", 1.0),
                         weight_decay=cfg.get_float("optimizer.weight_decay", 0.0), backend="b200",
                         deviation_every=cfg.get_int("train.deviation_every", 0), straggler=straggler)
    epochs = cfg.get_int("train.epochs", 0)
    steps_per_epoch = train_ds.n // batch_size
    total_steps = cfg.get_int("train.steps", epochs * steps_per_epoch)
    rows = []
    t0 = time.monotonic()
    if epochs > 0:
        for epoch in range(epochs):
            engine.run(steps_per_epoch)
            tl, ta = evaluate(model, train_ds)
            row = {"epoch": epoch, "train_loss": tl, "train_accuracy": ta, "test_loss": float("nan"),
                   "test_accuracy": float("nan"), "wall_time_s": time.monotonic() - t0}
            if test_ds is not None:
                row["test_loss"], row["test_accuracy"] = evaluate(model, test_ds)
            rows.append(row)
    else:
        engine.run(total_steps)
    log = engine.log
    log.to_jsonl(out / "train_log.jsonl")
    with open(out / "summary.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["epoch", "train_loss", "test_loss", "test_accuracy", "wall_time_s"])
        for r in rows:
            w.writerow([r["epoch"], f"{r['train_loss']:.9g}", f"{r['test_loss']:.9g}", f"{r['test_accuracy']:.9g}",
                        f"{r['wall_time_s']:.3f}"])
    result = {"steps": int(epochs * steps_per_epoch if epochs > 0 else total_steps), "epochs": epochs,
              "records": len(log.records), "checksum": log.checksum(), "epoch_rows": rows,
              "artifacts": {"train_log": str(out / "train_log.jsonl"), "summary": str(out / "summary.csv"),
                            "resolved_config": str(out / "resolved.cfg")}}
    if rows:
        result["final_train_loss"] = rows[-1]["train_loss"]
        result["final_train_accuracy"] = rows[-1]["train_accuracy"]
    dev_rows = engine.deviation_rows()
    if dev_rows:
        l_hat, m_hat = estimate_constants(dev_rows)
        report = lemma1_report(dev_rows, l_hat, m_hat)
        report["constants_source"] = "empirical_maxima"
        (out / "lemma_report.json").write_text(json.dumps(report, indent=2) + "\n")
        result["lemma_holds_fraction"] = report["holds_fraction"]
        result["artifacts"]["lemma_report"] = str(out / "lemma_report.json")
    (out / "resolved.cfg").write_text(render_config(cfg.raw))
    meta = {"schema_version": SCHEMA_VERSION, "kind": "train", "backend": "b200", "checksum": result["checksum"],
            "records": result["records"]}
    (out / "run_meta.json").write_text(json.dumps(meta, indent=2) + "\n")
    return result
