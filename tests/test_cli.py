"""CLI mirror (reference cli.py): option/config handling and exit codes on CPU; solve/train/bench on the GPU."""
import pytest

from paper_2602_02016_b200 import cli


def test_usage_errors_and_exit_codes(tmp_path, capsys):
    assert cli.main(["balance", "--workers", "2"]) == 1
    assert cli.main(["train", "--bogus", "1"]) == 1
    assert cli.main(["scalar-sweep"]) == 1
    bad = tmp_path / "bad.cfg"
    bad.write_text("nonsense_key = 3\n")
    assert cli.main(["train", "--config", str(bad)]) == 1
    assert cli.main(["balance", "--workers", "2", "--layers", str(tmp_path / "missing.txt")]) == 3
    layers = tmp_path / "l.txt"
    layers.write_text("0 5\n1 oops\n")
    assert cli.main(["balance", "--workers", "2", "--layers", str(layers)]) == 3


def test_balance_matches_reference_format(tmp_path, capsys):
    layers = tmp_path / "l.txt"
    layers.write_text("# id params\n0 5\n1 9\n2 5\n3 1\n4 9\n")
    out = tmp_path / "o.csv"
    assert cli.main(["balance", "--workers", "2", "--layers", str(layers), "--out", str(out)]) == 0
    assert out.read_text() == "worker,layer_id,params\n0,1,9\n0,0,5\n0,3,1\n1,4,9\n1,2,5\n"
    err = capsys.readouterr().err
    assert "# makespan = 15.0" in err and "# command = balance" in err


def test_config_precedence(tmp_path):
    import argparse

    cfg = tmp_path / "c.cfg"
    cfg.write_text("steps = 7\nblock_size = 32\n")
    args = cli._parser().parse_args(["train", "--config", str(cfg), "--steps", "3"])
    eff = cli.effective_config("train", args)
    assert eff["steps"] == 3 and eff["block-size"] == 32 and eff["lr"] == 0.1  # flag > file > default


@pytest.mark.gpu
def test_solve_train_bench_on_gpu(tmp_path, capsys):
    import numpy as np
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2602_02016_b200.linalg import format_matrix
    from paper_2602_02016_b200.tasks import random_spd

    m = tmp_path / "a.txt"
    m.write_text(format_matrix(random_spd(48, 50.0, seed=2)))
    out = tmp_path / "solve.txt"
    for method, p in (("ndb", 4), ("cn", 2), ("cbshv", 4), ("evd", 2)):
        assert cli.main(["solve", "--matrix", str(m), "--method", method, "--p", str(p), "--fixed-iters", "30",
                         "--out", str(out)]) == 0
        vals = dict(line.split(" = ") for line in out.read_text().splitlines())
        # degree-60 Chebyshev is itself inaccurate at the small eigenvalues: the reference reports 9.35e-2 here
        assert float(vals["oracle_rel_error"]) < (1e-3 if method != "cbshv" else 0.12), (method, vals)
    asym = tmp_path / "asym.txt"
    asym.write_text(format_matrix(np.triu(random_spd(8, 5.0, seed=1))))
    assert cli.main(["solve", "--matrix", str(asym)]) == 2
    tr = tmp_path / "train.csv"
    assert cli.main(["train", "--task", "logreg", "--steps", "5", "--block-size", "8", "--fixed-iters", "10",
                     "--lr", "0.5", "--out", str(tr)]) == 0
    lines = tr.read_text().splitlines()
    assert lines[0] == "step,loss,grad_norm,update_norm,refresh_flag" and len(lines) == 6
    assert float(lines[-1].split(",")[1]) < float(lines[1].split(",")[1])  # loss decreases
    be = tmp_path / "bench.csv"
    assert cli.main(["bench", "--batch", "4", "--dim", "64", "--repeats", "1", "--method", "ndb", "--p", "4",
                     "--out", str(be)]) == 0
    rows = be.read_text().splitlines()
    assert rows[0] == "mode,batch,dim,median_seconds,max_block_delta" and float(rows[1].split(",")[4]) < 1e-4
