"""Config / layer grammar of the run front door (runners.py) vs the reference's config.py."""

import pytest

import paper_1909_02625_b200 as P
from paper_1909_02625_b200.runners import ConfigParseError, RunConfig, parse_config_text, parse_layers, render_config, \
    run_validate


def test_reference_layer_grammar(stalepipe):
    from stalepipe.config import parse_layers as ref_parse

    for text in ["dense(12,16), relu, dense(16,12), tanh, dense(12,4)", "dense(6,16,false),relu,dense(16,3, true)"]:
        mine, ref = parse_layers(text), ref_parse(text)
        assert [(s.kind, s.in_dim, s.out_dim, s.bias) for s in mine] == \
            [(s.kind, s.in_dim, s.out_dim, s.bias) for s in ref]


def test_cnn_macros_and_errors():
    layers = parse_layers("resnet_cifar(20, 10)")
    assert layers == P.resnet_cifar_layers(20, 10)
    assert parse_layers("resnet_cifar_bottleneck(164,100)") == P.resnet_cifar_bottleneck_layers(164, 100)
    for bad in ["", "conv(3)", "dense(1)", "dense(a,b)"]:
        with pytest.raises(ConfigParseError):
            parse_layers(bad)


def test_config_text_roundtrip_and_validate(stalepipe):
    from stalepipe.config import parse_config_text as ref_parse_text, render_config as ref_render

    text = "# run\npipeline.p = 1,1,0\npipeline.m = 4,2,0\nmodel.layers = dense(12,16), relu, dense(16,4)\n"
    assert parse_config_text(text) == ref_parse_text(text)
    assert render_config(parse_config_text(text)) == ref_render(ref_parse_text(text))
    v = run_validate(RunConfig(parse_config_text(text)))
    assert v["q"] == [0, 1, 1] and v["staleness"] == [4, 2, 0] and v["max_staleness"] == 4
    with pytest.raises(ConfigParseError):
        parse_config_text("no equals sign")


def test_auto_boundaries():
    cfg = RunConfig({"pipeline.p": "1,1,1,0", "pipeline.m": "6,4,2,0", "model.layers": "resnet_cifar(56,10)",
                     "model.boundaries": "auto"})
    m = cfg.build_model()
    assert m.k == 4 and m.boundaries == P.flop_balanced_boundaries(P.resnet_cifar_layers(56, 10), 4)


SERVICE_CFG = {"pipeline.p": "1,1,0", "pipeline.m": "4,2,0",
               "model.layers": "dense(12,16), relu, dense(16,12), relu, dense(12,4)", "model.boundaries": "2,4",
               "data.source": "teacher", "data.teacher_dims": "12,8,4", "data.n_train": "64", "data.batch_size": "16",
               "optimizer.rule": "sum", "optimizer.lr": "0.05", "train.epochs": "1"}


def test_service_front_door_without_gpu():
    """The reference service's /health, /validate, /train (service.py:98-127) with train.backend = b200:
    a valid config validates, a bad one is a 400 naming the violated constraint, and /train on a box
    without a CUDA device is a 503 (no CPU fallback), never a silent CPU run."""
    import torch
    from fastapi.testclient import TestClient

    from paper_1909_02625_b200.service import create_app

    c = TestClient(create_app())
    assert c.get("/health").json()["backend"] == "b200"
    r = c.post("/validate", json={"config": SERVICE_CFG})
    assert r.status_code == 200 and r.json()["q"] == [0, 1, 1] and r.json()["max_staleness"] == 4
    r = c.post("/validate", json={"config": SERVICE_CFG, "overrides": {"pipeline.m": "2,1,0"}})
    assert r.status_code == 400 and "m[0]-p[0]-m[1] = 2-1-1 = 0" in r.json()["detail"]
    if not torch.cuda.is_available():
        r = c.post("/train", json={"config": SERVICE_CFG})
        assert r.status_code == 503 and "CUDA" in r.json()["detail"]
