"""The product TrainEngine's host logic (FIFOs, prefill tags, warmup policy, log,
multi-rank exchange) checked bitwise against the oracle engine on CPU.

The device runtime is swapped for tests/oracle_runtime.OracleRuntime (float64
oracle math), so every difference would come from the engine's schedule.
Multi-rank: world_size 2 over gloo on 127.0.0.1, blocks placed on both ranks,
cross-rank edges carried by TorchDistTransport (the same code NCCL runs).
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle.dsp_ref as R
import paper_1909_02625_b200 as P
from paper_1909_02625_b200.transport import LocalTransport
from tests.gpu_util import to_oracle_layers
from tests.oracle_runtime import OracleRuntime


def _layers():
    return [P.dense(12, 16), P.relu(), P.dense(16, 12), P.relu(), P.dense(12, 8), P.tanh(), P.dense(8, 4)]


def _cnn_layers():
    shape = (3, 6, 6)
    return [P.conv_bn_relu(shape, 4), P.basic_unit((4, 6, 6), 4, 1), P.basic_unit((4, 6, 6), 8, 2),
            P.avgpool((8, 3, 3)), P.dense(8, 5)]


def _oracle_run(layers, bounds, cfg_args, pool, steps, **kw):
    om = R.build_model(to_oracle_layers(layers), bounds)
    R.init_params(om, 7)
    eng = R.Engine(om, R.validate_config(*cfg_args[:2], warmup=cfg_args[2]), R.cycle(pool),
                   R.LrSchedule(0.05, ((steps // 2, 0.3),)), **kw)
    eng.run(steps)
    return eng, om


def _engine(layers, bounds, cfg_args, pool, steps, placement=None, transport=None, local=None, **kw):
    pm = P.build_model(layers, bounds)
    om = R.build_model(to_oracle_layers(layers), bounds)
    R.init_params(om, 7)
    K = pm.k
    local = local if local is not None else list(range(K))
    rt = OracleRuntime(om, local, pool[0][0].shape[0], rule=kw.get("rule", "sgd"), beta=kw.get("beta", 0.0),
                       s=kw.get("s", 1.0), weight_decay=kw.get("weight_decay", 0.0))
    eng = P.TrainEngine(pm, P.validate_config(*cfg_args[:2], warmup=cfg_args[2]), R.cycle(pool),
                        P.LrSchedule(0.05, ((steps // 2, 0.3),)), placement=placement, _runtime=rt,
                        _transport=transport or LocalTransport(), **kw)
    return eng, om


CASES = [
    ((1, 1, 1, 0), (6, 4, 2, 0), "faithful_zero_updates"),
    ((2, 2, 1, 0), (9, 5, 2, 0), "discard_warmup_updates"),
    ((1, 1, 1, 0), (7, 4, 2, 0), "faithful_zero_updates"),
]


@pytest.mark.parametrize("cfg", CASES)
def test_engine_schedule_bitwise_vs_oracle(cfg):
    pool = R.synthetic_batches(5, 6, (12, 1, 1), 4, seed=3)
    layers = _layers()
    bounds = [2, 4, 6]
    kw = dict(rule="sum", beta=0.9, s=0.8, weight_decay=1e-3)
    ref, om_ref = _oracle_run(layers, bounds, cfg, pool, 25, **kw)
    eng, om = _engine(layers, bounds, cfg, pool, 25, **kw)
    eng.run(10)
    eng.run(15)  # resumable: queue contents persist across run() calls
    assert eng.log.checksum() == ref.checksum()
    assert np.array_equal(om.flat_params(), om_ref.flat_params())
    assert eng.realized_staleness() == list(cfg[1])
    assert [r.loss is not None for r in eng.log.sorted()] == [r.block == 3 for r in eng.log.sorted()]


def test_engine_cnn_bitwise_vs_oracle():
    pool = R.synthetic_batches(4, 4, (3, 6, 6), 5, seed=2)
    cfg = ((1, 0), (2, 0), "faithful_zero_updates")
    ref, om_ref = _oracle_run(_cnn_layers(), [2], cfg, pool, 8, rule="sum", beta=0.9)
    eng, om = _engine(_cnn_layers(), [2], cfg, pool, 8, rule="sum", beta=0.9)
    eng.run(8)
    assert eng.log.checksum() == ref.checksum()
    assert np.array_equal(om.flat_params(), om_ref.flat_params())


def test_engine_rejects_cpu_backends_and_bad_placement():
    pool = R.synthetic_batches(2, 4, (12, 1, 1), 4, seed=3)
    pm = P.build_model(_layers(), [2, 4, 6])
    with pytest.raises(ValueError, match="backend"):
        P.TrainEngine(pm, P.validate_config((1, 1, 1, 0), (6, 4, 2, 0)), R.cycle(pool), P.LrSchedule(0.1),
                      backend="serial")
    with pytest.raises(P.ConfigError):
        P.TrainEngine(pm, P.validate_config((1, 0), (2, 0)), R.cycle(pool), P.LrSchedule(0.1))
    om = R.build_model(to_oracle_layers(_layers()), [2, 4, 6])
    with pytest.raises(P.ConfigError, match="placement"):
        P.TrainEngine(pm, P.validate_config((1, 1, 1, 0), (6, 4, 2, 0)), R.cycle(pool), P.LrSchedule(0.1),
                      placement=[0, 0, 1, 1], _runtime=OracleRuntime(om, [0, 1], 4), _transport=LocalTransport())


# ------------------------------------------------------------------ world_size 2 (gloo)
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, placement, cfg, out_dir, layers_name):
    import torch.distributed as dist

    from paper_1909_02625_b200.transport import TorchDistTransport

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layers = _layers() if layers_name == "mlp" else _cnn_layers()
        bounds = [2, 4, 6] if layers_name == "mlp" else [1, 2, 3]
        shape = (12, 1, 1) if layers_name == "mlp" else (3, 6, 6)
        pool = R.synthetic_batches(5, 6, shape, 4, seed=3)
        local = [k for k, r in enumerate(placement) if r == rank]
        eng, om = _engine(layers, bounds, cfg, pool, 20, placement=placement, transport=TorchDistTransport(),
                          local=local, rule="sum", beta=0.9, weight_decay=1e-3)
        eng.run(12)
        eng.run(8)
        recs = [(r.step, r.block, r.batch_index, r.loss, r.grad_norm) for r in eng.log.sorted()]
        params = {k: om.blocks[k].params for k in local}
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.array([recs, params], dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("placement,layers_name", [([0, 0, 1, 1], "mlp"), ([0, 1, 0, 1], "mlp"),
                                                    ([1, 0, 0, 1], "cnn")])
def test_two_rank_pipeline_bitwise_vs_single_process(placement, layers_name):
    cfg = ((1, 1, 1, 0), (6, 4, 2, 0), "faithful_zero_updates")
    layers = _layers() if layers_name == "mlp" else _cnn_layers()
    bounds = [2, 4, 6] if layers_name == "mlp" else [1, 2, 3]
    shape = (12, 1, 1) if layers_name == "mlp" else (3, 6, 6)
    pool = R.synthetic_batches(5, 6, shape, 4, seed=3)
    ref, om_ref = _oracle_run(layers, bounds, cfg, pool, 20, rule="sum", beta=0.9, weight_decay=1e-3)
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), placement, cfg, d, layers_name), nprocs=2, join=True,
                           start_method="spawn")
        recs, params = [], {}
        for rank in range(2):
            rr, pp = np.load(os.path.join(d, f"rank{rank}.npy"), allow_pickle=True)
            recs += rr
            params.update(pp)
    recs.sort(key=lambda r: (r[0], r[1]))
    want = sorted(((r.step, r.block, r.batch_index, r.loss, r.grad_norm) for r in ref.records),
                  key=lambda r: (r[0], r[1]))
    assert recs == want
    for k in range(4):
        assert np.array_equal(params[k], om_ref.blocks[k].params)


def _stall_worker(rank, world, port, out_dir):
    """Rank 1 never reaches the exchange within the watchdog: rank 0 must raise DeadlockError
    with the reference's message (pipeline.py:644-657), not hang."""
    import time

    import torch.distributed as dist

    from paper_1909_02625_b200.transport import TorchDistTransport

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    layers = _layers()
    pool = R.synthetic_batches(5, 6, (12, 1, 1), 4, seed=3)
    placement = [0, 0, 1, 1]
    local = [k for k, r in enumerate(placement) if r == rank]
    cfg = ((1, 1, 1, 0), (6, 4, 2, 0), "faithful_zero_updates")
    eng, _ = _engine(layers, [2, 4, 6], cfg, pool, 20, placement=placement, transport=TorchDistTransport(),
                     local=local, rule="sgd", watchdog_s=1.0)
    if rank == 1:
        time.sleep(4.0)
        with open(os.path.join(out_dir, "rank1.txt"), "w") as f:
            f.write("slept")
        os._exit(0)  # a dead peer
    try:
        eng.run(2)
        res = "no error"
    except P.DeadlockError as e:
        res = "DeadlockError: " + str(e)
    with open(os.path.join(out_dir, "rank0.txt"), "w") as f:
        f.write(res)
    os._exit(0)


def test_two_rank_watchdog_raises_deadlock_error():
    with tempfile.TemporaryDirectory() as d:
        ctx = mp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=_stall_worker, args=(r, 2, port, d)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(60)
            if p.is_alive():
                p.kill()
        res = open(os.path.join(d, "rank0.txt")).read()
    assert res.startswith("DeadlockError: workers stalled after 1.0s; queue occupancy"), res
    assert "steps" in res
