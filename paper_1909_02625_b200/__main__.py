"""CLI: ``python -m paper_1909_02625_b200 {validate,train} --config RUN.cfg [--out DIR] [--set k=v ...]``.

The reference's ``stalepipe validate`` / ``stalepipe train`` (cli.py:103-119) on the B200
engine: same config files, ``train.backend = b200``.
"""

import argparse
import json
import sys

from .runners import RunConfig, load_config_file, run_train, run_validate


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1909_02625_b200")
    ap.add_argument("command", choices=["validate", "train"])
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", default="runs/b200")
    ap.add_argument("--set", action="append", default=[], metavar="KEY=VALUE", help="override a config key")
    args = ap.parse_args(argv)
    raw = load_config_file(args.config)
    for kv in args.set:
        k, _, v = kv.partition("=")
        raw[k.strip()] = v.strip()
    raw.setdefault("train.backend", "b200")
    cfg = RunConfig(raw)
    res = run_validate(cfg) if args.command == "validate" else run_train(cfg, args.out)
    print(json.dumps(res, indent=2, default=float))
    return 0


if __name__ == "__main__":
    sys.exit(main())
