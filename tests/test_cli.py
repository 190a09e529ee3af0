"""The command-line outputs (SPEC.md cli module): config parsing diagnostics on CPU; a
full run / compare / memory-audit on the GPU."""
import csv
import os

import pytest

from paper_2404_01407_b200.cli import ConfigParseError, main, parse_config, read_kv


def test_config_parse_and_diagnostics():
    c = parse_config("# c1 run\ncase = c1\nscale = 0.25  # small\nmode = explicit\nmg_levels = 2\n")
    assert c == dict(case="c1", scale=0.25, mode="explicit", mg_levels=2)
    with pytest.raises(ConfigParseError, match=r"cfg:2: unknown key 'cells'"):
        parse_config("case = c1\ncells = 4\n", "cfg")
    with pytest.raises(ConfigParseError, match=r"cfg:1: key 'scale'"):
        parse_config("scale = big\n", "cfg")
    with pytest.raises(ConfigParseError, match="missing required key 'case'"):
        parse_config("scale = 0.5\n", "cfg")
    with pytest.raises(ConfigParseError, match="expected 'key = value'"):
        parse_config("case c1\n", "cfg")


def test_config_errors_exit_2(tmp_path, capsys):
    p = tmp_path / "bad.cfg"
    p.write_text("scale = 0.5\n")
    assert main(["run", str(p), "--out", str(tmp_path / "o")]) == 2
    assert "missing required key 'case'" in capsys.readouterr().err
    assert main(["run", "c1", "--mode", "implicit", "--mg-levels", "2", "--out", str(tmp_path / "o")]) == 2


@pytest.mark.gpu
def test_run_compare_bench(tmp_path):
    cfg = tmp_path / "c1.cfg"
    cfg.write_text("case = c1\nscale = 0.25\nharmonics = 2\nmax_iters = 6\n")
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    assert main(["run", str(cfg), "--out", a, "--fields"]) == 3  # iteration cap
    assert main(["run", str(cfg), "--out", b, "--fields"]) == 3
    with open(os.path.join(a, "convergence.csv")) as f:
        rows = list(csv.reader(f))
    assert rows[0] == ["iter", "resid_mean", "resid_h0", "resid_h1", "R_z", "seconds", "WU"]
    assert len(rows) == 7
    man, summ = read_kv(os.path.join(a, "manifest.txt")), read_kv(os.path.join(a, "summary.txt"))
    assert man["mode"] == "implicit" and float(man["cfl"]) == 10.0 and float(man["t_ref_seconds"]) > 0
    assert summ["reason"] == "iteration-cap" and summ["iterations"] == "6" and summ["exit_code"] == "3"
    # determinism: same manifest -> bitwise identical convergence CSV; self-compare passes
    with open(os.path.join(b, "convergence.csv")) as f:
        rows_b = list(csv.reader(f))
    assert [r[:5] for r in rows] == [r[:5] for r in rows_b]
    assert main(["compare", a, b, "--bound", "0"]) == 0
    assert main(["run", "c1", "--scale", "0.25", "--harmonics", "2", "--max-iters", "40", "--target-drop", "2",
                 "--out", str(tmp_path / "t")]) == 0
    assert main(["compare", a, str(tmp_path / "t")]) == 2  # harmonics / scale mismatch or no fields
    out = str(tmp_path / "mem.csv")
    assert main(["bench", "memory-audit", "--out", out]) == 0
    with open(out) as f:
        mem = list(csv.DictReader(f))
    assert len({r["peak_lhs_bytes"] for r in mem}) == 1


@pytest.mark.gpu
def test_oracle_command(tmp_path):
    """`oracle`: FNLH run + the time-accurate march; fields in the run layout (so `compare`
    applies between a run and its oracle), amplitude errors on interior nodes."""
    o, a = str(tmp_path / "o"), str(tmp_path / "a")
    args = ["c1", "--scale", "0.5", "--harmonics", "1", "--max-iters", "400", "--target-drop", "8", "--tol", "0.01",
            "--sweeps", "10"]
    assert main(["oracle"] + args + ["--out", o]) in (0, 3)
    summ = read_kv(os.path.join(o, "summary.txt"))
    assert summ["periodic"] == "1" and float(summ["amp_error_h0"]) < 0.02
    with open(os.path.join(o, "amplitude_errors.csv")) as f:
        rows = list(csv.DictReader(f))
    assert len(rows) == 1 and float(rows[0]["rel_l2_interior"]) < 0.02
    assert main(["run"] + args + ["--out", a, "--fields"]) in (0, 3)
    assert main(["compare", a, o, "--bound", "0.05"]) == 0
