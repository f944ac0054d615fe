"""PSAT files (tensorfile.py:23-78) against bytes written by the real reference
(tests/golden/psat_files.npz), their error taxonomy (test_acceptance.py:265-290 cases), and the
pyrattn-compatible command line (cli.py:39-62, exit codes :21-24)."""

import json
import struct

import numpy as np
import pytest

from helpers import GOLDEN_DIR


def test_write_matches_reference_bytes_and_read_round_trips(tmp_path):
    from paper_2512_04025_b200.tensorfile import read_tensor, write_tensor
    z = np.load(GOLDEN_DIR / "psat_files.npz")
    i = 0
    while f"in{i}" in z:
        path = tmp_path / f"t{i}.psat"
        write_tensor(path, z[f"in{i}"])
        assert path.read_bytes() == z[f"bytes{i}"].tobytes()
        ref_file = tmp_path / f"r{i}.psat"
        ref_file.write_bytes(z[f"bytes{i}"].tobytes())
        got = read_tensor(ref_file)
        assert got.dtype == np.float64 and got.shape == z[f"read{i}"].shape
        assert np.array_equal(got, z[f"read{i}"])
        i += 1
    assert i == 4


def test_malformed_files_raise_tensor_file_error(tmp_path):
    from paper_2512_04025_b200.errors import TensorFileError, ValidationError
    from paper_2512_04025_b200.tensorfile import read_tensor, write_tensor
    bad = tmp_path / "bad.psat"
    cases = [(b"PSA", "truncated header"), (b"NOPE" + struct.pack("<II", 1, 1), "magic"),
             (b"PSAT" + struct.pack("<II", 9, 1), "version"),
             (b"PSAT" + struct.pack("<II", 1, 9), "ndims"),
             (b"PSAT" + struct.pack("<II", 1, 2) + struct.pack("<Q", 3), "dimension list"),
             (b"PSAT" + struct.pack("<II", 1, 1) + struct.pack("<Q", 0), "zero-length"),
             (b"PSAT" + struct.pack("<II", 1, 1) + struct.pack("<Q", 4) + b"\0" * 12,
              "truncated payload"),
             (b"PSAT" + struct.pack("<II", 1, 1) + struct.pack("<Q", 1) + b"\0" * 8, "trailing"),
             (b"PSAT" + struct.pack("<II", 1, 1) + struct.pack("<Q", 1)
              + struct.pack("<f", float("nan")), "NaN")]
    for blob, word in cases:
        bad.write_bytes(blob)
        with pytest.raises(TensorFileError, match=word):
            read_tensor(bad)
    for arr in (np.zeros(0), np.array([np.inf]), np.zeros((1,) * 9)):
        with pytest.raises(ValidationError):
            write_tensor(tmp_path / "w.psat", arr)


def test_cli_report_and_error_exit_codes(tmp_path, capsys):
    from paper_2512_04025_b200.cli import main
    rep = {"heads": 2, "relative_error": 0.01, "schedule_relative_error": 0.01,
           "sparsity": {"rho_bar": 0.2, "sparsity": 0.5, "kv_coverage": 0.6,
                        "level_histogram": [1, 2]},
           "utilization": {"tiles": 3, "utilization": 0.9}, "skipped_rows": 0,
           "wall_time_s": 0.5}
    path = tmp_path / "r.json"
    path.write_text(json.dumps(rep))
    assert main(["report", "--in", str(path)]) == 0
    assert "effective budget rho:  0.2000" in capsys.readouterr().out
    assert main(["report", "--in", str(path), "--csv"]) == 0
    assert "sparsity.rho_bar,0.2" in capsys.readouterr().out
    path.write_text("{}")
    assert main(["report", "--in", str(path)]) == 2
    cfg = tmp_path / "c.json"
    cfg.write_text("{not json")
    assert main(["run", "--config", str(cfg), "--q", "a", "--k", "b", "--v", "c"]) == 2
    cfg.write_text(json.dumps({"n": 128, "d": 16, "b_q": 64, "b_k": 64, "levels": 2,
                               "estimator": "sampled-max", "s_q": 4, "s_k": 4, "seed": 0,
                               "mask": "threshold", "thresholds": [0.5, 0.9], "tile_len": 64}))
    assert main(["run", "--config", str(cfg), "--q", str(tmp_path / "missing.psat"),
                 "--k", "b", "--v", "c"]) == 3


@pytest.mark.gpu
def test_cli_run_matches_run_pipeline(tmp_path, capsys):
    """`run` on PSAT files = run_pipeline on the same arrays (report fields and output)."""
    import paper_2512_04025_b200 as psa
    from paper_2512_04025_b200.cli import main
    from paper_2512_04025_b200.tensorfile import read_tensor, write_tensor
    rng = np.random.default_rng(8)
    names = {}
    for name in ("q", "k", "v"):
        names[name] = tmp_path / f"{name}.psat"
        write_tensor(names[name], rng.standard_normal((2, 1024, 64)))
    conf = {"n": 1024, "d": 64, "b_q": 64, "b_k": 64, "levels": 4, "estimator": "sampled-max",
            "s_q": 8, "s_k": 8, "seed": 0, "mask": "threshold",
            "thresholds": [0.164713, 0.282366, 0.376488, 0.95], "tile_len": 128}
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps(conf))
    out_rep, out_t = tmp_path / "rep.json", tmp_path / "o.psat"
    rc = main(["run", "--config", str(cfg), "--q", str(names["q"]), "--k", str(names["k"]),
               "--v", str(names["v"]), "--out", str(out_rep), "--out-tensor", str(out_t)])
    assert rc == 0
    rep = json.loads(out_rep.read_text())
    res = psa.run_pipeline(psa.RunConfig.from_dict(conf), *(read_tensor(names[x]) for x in "qkv"))
    for key in ("heads", "sparsity", "utilization", "skipped_rows", "steps", "config"):
        assert rep[key] == res.report[key]
    o = read_tensor(out_t)
    assert o.shape == (2, 1024, 64)
    assert np.array_equal(o, res.output.astype(np.float32).astype(np.float64))
