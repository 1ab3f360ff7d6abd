"""``restore`` on the GPU path: a reference restore config runs unchanged.

    python -m paper_2002_02328_b200.restore --config restore.cfg [--override key=value ...]

Same flat key=value config as the reference CLI (reference cli.py:60-70
schema, :94-138 parser, :200-217 cmd_restore, :296-327 exit codes 0 / 1
configuration or format error / 2 runtime abort), with one optional extra
key, ``dtype`` (f64 default, or f32 for the device arithmetic).  The
observation streams from its BD3MGVOL file straight into device memory
(volume.read_volume(..., device=)), the solve runs through runtime.run on
the CUDA kernels, and the outputs (restored volume, log CSV, trace CSV) are
written in the reference's formats.  Only the restore command is mirrored:
phantom / degrade / ablate / speedup are experiment drivers, out of scope.
"""

from __future__ import annotations

import argparse
import sys

from . import blur, runtime, scheduler
from .objective import Objective, RegParams
from .volume import FormatError, init_uniform, read_volume, snr_db, write_volume


class ConfigError(Exception):
    pass


_SCHEMA = {  # reference cli.py:29-45, :71-80 (restore)
    "observed": ("s", True, None), "psf": ("s", True, None), "out": ("s", True, None),
    "method": ("s", True, None), "workers": ("i", True, None),
    "truth": ("s", False, None), "log_out": ("s", False, None), "trace_out": ("s", False, None),
    "max_updates": ("i", False, None),
    "block_height": ("i", False, 1), "tol": ("f", False, 1e-6), "engine": ("s", False, "simulated"),
    "init_seed": ("i", False, 0), "run_seed": ("i", False, 0), "cg_tol": ("f", False, 1e-8),
    "cg_maxit": ("i", False, 200),
    "lambda": ("f", False, 0.1), "eta": ("f", False, 1.0), "kappa": ("f", False, 0.05),
    "delta": ("f", False, 0.05), "x_min": ("f", False, 0.0), "x_max": ("f", False, 1.0),
    "dtype": ("s", False, "f64"),
}


def _parse_pairs(lines, where) -> dict[str, str]:
    pairs = {}
    for ln, raw in enumerate(lines, 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"{where}:{ln}: expected key=value, got {line!r}")
        key, value = (part.strip() for part in line.split("=", 1))
        if not key:
            raise ConfigError(f"{where}:{ln}: empty key")
        pairs[key] = value
    return pairs


def load_config(path: str, overrides: list[str]) -> dict:
    try:
        with open(path) as fh:
            pairs = _parse_pairs(fh, path)
    except OSError as exc:
        raise ConfigError(f"cannot read config {path}: {exc}") from exc
    pairs.update(_parse_pairs(overrides, "--override"))
    cfg = {}
    for key, value in pairs.items():
        if key not in _SCHEMA:
            raise ConfigError(f"unknown config key: {key}")
        kind = _SCHEMA[key][0]
        try:
            cfg[key] = int(value) if kind == "i" else float(value) if kind == "f" else value
        except ValueError as exc:
            raise ConfigError(f"key {key}: cannot parse {value!r} as "
                              f"{'integer' if kind == 'i' else 'number'}") from exc
    for key, (_, required, default) in _SCHEMA.items():
        if key not in cfg:
            if required:
                raise ConfigError(f"missing required key: {key}")
            cfg[key] = default
    if cfg["dtype"] not in ("f64", "f32"):
        raise ConfigError(f"key dtype: expected f64 or f32, got {cfg['dtype']!r}")
    return cfg


def cmd_restore(cfg) -> int:
    import torch

    dt = torch.float64 if cfg["dtype"] == "f64" else torch.float32
    y = read_volume(cfg["observed"], device="cuda", dtype=dt)
    psf = blur.read_psf(cfg["psf"])
    reg = RegParams(lam=cfg["lambda"], eta=cfg["eta"], kappa=cfg["kappa"], delta=cfg["delta"],
                    x_min=cfg["x_min"], x_max=cfg["x_max"])
    obj = Objective(psf, y, reg)
    truth = read_volume(cfg["truth"]) if cfg["truth"] else None
    x0 = init_uniform(obj.dims, max(0.0, float(obj.y.max())), cfg["init_seed"])  # cli.py:152-156
    run_cfg = runtime.RunConfig(method=cfg["method"], workers=cfg["workers"], block_height=cfg["block_height"],
                                tol=cfg["tol"], max_updates=cfg["max_updates"], seed=cfg["run_seed"],
                                cg_tol=cfg["cg_tol"], cg_maxit=cfg["cg_maxit"], engine=cfg["engine"],
                                dtype=cfg["dtype"])
    result = runtime.run(obj, x0, run_cfg, truth=truth)
    write_volume(result.x_final, cfg["out"])
    if cfg["log_out"]:
        runtime.write_log_csv(result.log, cfg["log_out"])
    if cfg["trace_out"]:
        scheduler.write_trace_csv(result.trace, cfg["trace_out"])
    print(f"final f = {result.log[-1].f_value:.10g}")
    if truth is not None:
        print(f"restored snr_db = {snr_db(truth, result.x_final):.4f}")
    print(f"tau_hat = {result.tau_hat}")
    print(f"stop_reason = {result.stop_reason}")
    return 0


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage problems are configuration errors
        raise ConfigError(message)


def main(argv=None) -> int:
    parser = _Parser(prog="bd3mg-restore", description=__doc__)
    parser.add_argument("--config", required=True)
    parser.add_argument("--override", action="append", default=[], metavar="KEY=VALUE")
    try:
        args = parser.parse_args(argv)
        return cmd_restore(load_config(args.config, args.override))
    except (ConfigError, FormatError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except Exception as exc:  # noqa: BLE001 -- reference cli.py:322-324
        print(f"abort: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
