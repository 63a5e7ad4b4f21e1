"""bench.py contract checks that need no GPU: the reference arm's JSON line (the CPU oracle of the
reference DSP step on a bounded sub-batch, its sub-batch stated in config) and the argument
surface the driver uses."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--model", "resnet56", "--steps", "1",
                          "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "samples/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["global_batch"] == 32 and d["config"]["workload_global_batch"] == 128
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1


def test_default_model_is_baseline_config4():
    sys.path.insert(0, ROOT)
    import bench

    sys_argv = sys.argv
    try:
        sys.argv = ["bench.py"]
        args = bench.parse()
    finally:
        sys.argv = sys_argv
    assert args.model == "resnet50" and args.gpus == 1
    assert bench.MODELS["resnet50"]["cfg"] == 4 and bench.MODELS["resnet50"]["batch"] == 256
    assert bench.roofline_spec("resnet50", 256)["bound"] == "tensor"
