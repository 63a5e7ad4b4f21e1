"""run_train with train.backend = b200 (runners.py): the reference's artifacts,
and the same log as a TrainEngine built by hand from the same config."""

import json

import numpy as np
import pytest

import paper_1909_02625_b200 as P
from paper_1909_02625_b200.rng import derive_seed
from paper_1909_02625_b200.runners import RunConfig, parse_config_text, run_train

pytestmark = pytest.mark.gpu

MLP = """
pipeline.p = 1,1,0
pipeline.m = 4,2,0
model.layers = dense(12,16), relu, dense(16,12), relu, dense(12,4)
model.boundaries = 2,4
data.source = teacher
data.teacher_dims = 12,8,4
data.n_train = 256
data.n_test = 64
data.batch_size = 16
optimizer.rule = sum
optimizer.lr = 0.05
optimizer.lr_decay_steps = 20
train.epochs = 2
train.seed = 3
"""


def test_run_train_mlp_artifacts_and_checksum(tmp_path):
    cfg = RunConfig(parse_config_text(MLP))
    res = run_train(cfg, tmp_path)
    for k in ("train_log", "summary", "resolved_config"):
        assert (tmp_path / res["artifacts"][k].split("/")[-1]).exists()
    assert res["steps"] == 2 * (256 // 16) and len(res["epoch_rows"]) == 2
    assert np.isfinite(res["final_train_loss"]) and 0.0 <= res["final_train_accuracy"] <= 1.0
    lines = (tmp_path / "train_log.jsonl").read_text().splitlines()
    assert json.loads(lines[0])["kind"] == "train_log" and len(lines) == 1 + res["records"]
    assert json.loads((tmp_path / "run_meta.json").read_text())["backend"] == "b200"
    # the same run through the oracle engine (bf16-storage emulation, fed the identical batches from
    # the data pipeline, which tests/test_host_cpu.py pins bitwise to the reference's epoch_stream):
    # schedule exact, losses within the bf16 tolerance of tests/test_engine_gpu.py
    import oracle.dsp_ref as R
    from tests.gpu_util import to_oracle_layers

    batches = P.epoch_stream(cfg.build_dataset("train"), 16, shuffle_seed=derive_seed(3, 1))
    from paper_1909_02625_b200.runners import parse_layers

    sched = cfg.build_schedule()
    with R.storage("bf16"):
        om = R.build_model(to_oracle_layers(parse_layers(cfg.get("model.layers"))), [2, 4])
        R.init_params(om, cfg.get_int("model.init_seed", cfg.get_int("train.seed", 0)))
        ref = R.Engine(om, R.validate_config((1, 1, 0), (4, 2, 0)), batches, R.LrSchedule(sched.base, sched.decays),
                       rule="sum", beta=0.9)
        ref.run(res["steps"])
    got = [json.loads(ln) for ln in lines[1:]]
    want = sorted(ref.records, key=lambda r: (r.step, r.block))
    assert [(g["step"], g["block"], g["batch_index"]) for g in got] == [(r.step, r.block, r.batch_index) for r in want]
    for g, r in zip(got, want):
        if r.loss is not None:
            assert abs(g["loss"] - r.loss) <= 1e-2 * max(1.0, abs(r.loss)), (g, r)


def test_service_train_matches_run_train(tmp_path):
    """POST /train (the reference service's train endpoint, service.py:118-127) runs the B200 engine:
    same checksum as run_train on the same config."""
    from fastapi.testclient import TestClient

    from paper_1909_02625_b200.service import create_app

    raw = parse_config_text(MLP)
    direct = run_train(RunConfig(dict(raw)), tmp_path / "direct")
    r = TestClient(create_app()).post("/train", json={"config": raw, "out_dir": str(tmp_path / "svc")})
    assert r.status_code == 200, r.text
    body = r.json()
    assert body["checksum"] == direct["checksum"] and body["records"] == direct["records"]
    assert len(body["epoch_rows"]) == 2


def test_run_train_cnn_with_deviation_report(tmp_path):
    raw = parse_config_text(MLP)
    raw.update({"model.layers": "resnet_cifar(8, 10, 8)", "model.boundaries": "auto", "data.source": "synthetic",
                "data.shape": "3,32,32", "data.classes": "10", "data.n_train": "64", "data.n_test": "32",
                "data.batch_size": "8", "train.epochs": "1", "train.deviation_every": "3"})
    res = run_train(RunConfig(raw), tmp_path)
    assert "lemma_report" in res["artifacts"]
    report = json.loads((tmp_path / "lemma_report.json").read_text())
    assert report["samples"] >= 1 and 0.0 <= report["holds_fraction"] <= 1.0


def test_cli_validate(tmp_path, capsys):
    from paper_1909_02625_b200.__main__ import main

    path = tmp_path / "run.cfg"
    path.write_text(MLP)
    assert main(["validate", "--config", str(path)]) == 0
    assert json.loads(capsys.readouterr().out)["q"] == [0, 1, 1]


def test_batch_width_mismatch_is_a_shape_error():
    """A batch whose width is not the model's input size is rejected (the reference's
    matmul shape check), never packed out of bounds."""
    model = P.build_model(P.resnet_cifar_layers(8, 10, width=8), [])
    P.init_params(model, 0)
    bad = [(np.zeros((4, 3 * 8 * 8)), np.zeros(4, dtype=np.int64))]
    eng = P.TrainEngine(model, P.validate_config((0,), (0,)), iter(bad * 2), P.LrSchedule(0.1))
    with pytest.raises(P.ShapeError):
        eng.run(1)
    ne = P.NativeEngine(model, P.validate_config((0,), (0,)), 4, P.LrSchedule(0.1))
    with pytest.raises(P.ShapeError):
        ne.run_batches(np.zeros((1, 4, 192)), np.zeros((1, 4), dtype=np.int64))
