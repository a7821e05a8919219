"""Command line (the reference's tools/biewos.cpp on the B200 path):

  python -m paper_1210_1491_b200 solve <config.cfg> [--set sec.key=v ...] [--seed N] [--workers N]
  python -m paper_1210_1491_b200 compare <a.csv> <b.csv> <tol>

Exit code 2 on any error (tools/biewos.cpp:52-55)."""
from __future__ import annotations

import argparse
import sys


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1210_1491_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve")
    s.add_argument("config")
    s.add_argument("--set", action="append", default=[])
    s.add_argument("--seed", type=int)
    s.add_argument("--workers", type=int)
    c = sub.add_parser("compare")
    c.add_argument("a")
    c.add_argument("b")
    c.add_argument("tol", type=float)
    args = ap.parse_args(argv)
    try:
        from . import runner

        if args.cmd == "compare":
            return runner.compare_csv(args.a, args.b, args.tol, sys.stdout)
        cfg = runner.parse_config_file(args.config)
        for spec in args.set:
            runner.apply_override(cfg, spec)
        rec = runner.run(cfg, seed=args.seed, workers=args.workers)
        runner.write_outputs(rec, cfg)
        sys.stderr.write(f"{rec.method}: {len(rec.rows)} rows, {rec.paths_total:.3g} paths, "
                         f"{rec.wall_seconds:.3f} s\n")
        if not runner.RawConfig.has(cfg, "output", "csv"):
            sys.stdout.write(rec.csv_text)
        return 0
    except Exception as e:  # noqa: BLE001 — the CLI contract: any failure -> exit 2
        sys.stderr.write(f"error: {type(e).__name__}: {e}\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
