"""The reference restore config on the GPU path (paper_2002_02328_b200.restore,
mirroring reference cli.py:94-138, :200-217, :296-327): config errors on CPU,
and an end-to-end restore on the GPU checked against the oracle."""

import csv

import numpy as np
import pytest

from paper_2002_02328_b200 import restore


def _write_cfg(path, **kv):
    path.write_text("# restore config\n" + "".join(f"{k} = {v}\n" for k, v in kv.items()))
    return str(path)


@pytest.mark.parametrize("extra, msg", [
    ({"bogus": 1}, "unknown config key: bogus"),
    ({"workers": "two"}, "cannot parse"),
    ({"dtype": "f16"}, "expected f64 or f32"),
])
def test_config_errors_exit_1(extra, msg, tmp_path, capsys):
    kv = dict(observed="y.vol", psf="h.psf", out="x.vol", method="bd3mg", workers=1)
    kv.update(extra)
    assert restore.main(["--config", _write_cfg(tmp_path / "c", **kv)]) == 1
    assert msg in capsys.readouterr().err


def test_missing_key_and_missing_file(tmp_path, capsys):
    assert restore.main(["--config", _write_cfg(tmp_path / "c", observed="y", psf="h", out="x", method="bd3mg")]) == 1
    assert "missing required key: workers" in capsys.readouterr().err
    assert restore.main(["--config", str(tmp_path / "nope")]) == 1
    assert "cannot read config" in capsys.readouterr().err


@pytest.mark.gpu
def test_restore_matches_oracle(tmp_path, oracle_mod, capsys):
    from paper_2002_02328_b200 import blur
    from paper_2002_02328_b200.volume import Dims3, init_uniform, read_volume, write_volume

    dims = Dims3(24, 20, 12)
    psf = blur.depth_variant_stack(dims, (3, 3, 5), (0.8, 1.6), (1.0, 2.0))
    rng = np.random.Generator(np.random.Philox(9))
    truth = rng.uniform(0, 1, dims.shape)
    y = oracle_mod.H(psf.kernels, truth) + 0.01 * rng.standard_normal(dims.shape)
    write_volume(y, tmp_path / "y.vol")
    blur.write_psf(psf, tmp_path / "h.psf")
    write_volume(truth, tmp_path / "t.vol")
    cfg = _write_cfg(tmp_path / "c", observed=tmp_path / "y.vol", psf=tmp_path / "h.psf", out=tmp_path / "x.vol",
                     truth=tmp_path / "t.vol", method="bd3mg", workers=1, block_height=4, tol=1e-30,
                     max_updates=9, log_out=tmp_path / "log.csv", trace_out=tmp_path / "trace.csv",
                     **{"lambda": 0.01, "eta": 0.1, "delta": 0.01})
    assert restore.main(["--config", cfg]) == 0
    out = capsys.readouterr().out
    assert "final f = " in out and "stop_reason = " in out and "restored snr_db" in out
    got = read_volume(tmp_path / "x.vol")
    crit = oracle_mod.Criterion(psf.kernels, y, lam=0.01, eta=0.1, kappa=0.05, delta=0.01)
    x0 = init_uniform(dims, max(0.0, float(y.max())), 0)
    want = oracle_mod.run_bd3mg(crit, x0, 1, 4, max_updates=9)[0]
    assert np.linalg.norm(got - want) <= 1e-9 * np.linalg.norm(want)
    rows = list(csv.reader(open(tmp_path / "log.csv")))
    assert rows[0] == ["k", "wall_seconds", "f", "snr_db", "rel_dist", "max_staleness"] and len(rows) >= 2
    assert len(list(csv.reader(open(tmp_path / "trace.csv")))) == 1 + 9
