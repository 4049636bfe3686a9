"""CLI `solve` (reference cli.py:119-255, tests/test_cli.py:20-122)."""

import json
import os

import pytest

from conftest import GOLDEN, gpu_available

from paper_2407_09848_b200.cli import EXIT_CONFIG, EXIT_OK, ConfigError, build_problem, main, parse_config


class TestConfigParsing:
    def test_defaults_without_file(self):
        cfg = parse_config(None, [])
        assert cfg["problem"] == "poisson3d"
        assert cfg["smoother"] == "opt_cheb1"

    def test_file_and_overrides(self, tmp_path):
        p = tmp_path / "run.cfg"
        p.write_text("# comment\nproblem = poisson3d_27\nm = 16\n")
        cfg = parse_config(str(p), ["m=32"])
        assert cfg["problem"] == "poisson3d_27" and cfg["m"] == "32"

    def test_unknown_key_rejected(self):
        with pytest.raises(ConfigError):
            parse_config(None, ["nonsense=1"])

    def test_malformed_line_rejected(self, tmp_path):
        p = tmp_path / "bad.cfg"
        p.write_text("this is not a key value pair\n")
        with pytest.raises(ConfigError):
            parse_config(str(p), [])

    def test_build_problem_dispatch(self):
        A, b = build_problem(parse_config(None, ["problem=poisson3d", "m=3"]))
        assert A.nrows == 27
        A, b = build_problem(parse_config(None, ["problem=poisson3d_27", "m=3"]))
        assert A.nnz == 7 ** 3
        with pytest.raises(ConfigError):
            build_problem(parse_config(None, ["problem=spectral"]))


def test_config_error_exit_code(capsys):
    assert main(["solve", "--override", "bogus=1"]) == EXIT_CONFIG
    assert main(["solve", "--override", "smoother=sor"]) == EXIT_CONFIG


CASES = {
    "cli_solve_m8_matching.json": ["m=8", "coarsening=pairwise_matching"],
    "cli_solve_m12_sa.json": ["m=12", "smoother=cheb4", "tol=1e-6"],
    "cli_solve_m6_itmax1.json": ["m=6", "itmax=1"],
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_solve_report_matches_reference_and_is_byte_identical(name, tmp_path, capsys):
    if not gpu_available():
        pytest.skip("no CUDA device")
    args = ["solve"] + [x for o in CASES[name] for x in ("--override", o)]
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    assert main(args + ["-o", str(a)]) == EXIT_OK
    assert main(args + ["-o", str(b)]) == EXIT_OK
    assert a.read_bytes() == b.read_bytes()  # deterministic device reductions
    got = json.loads(a.read_text())
    with open(os.path.join(GOLDEN, name)) as f:
        want = json.load(f)
    assert got["config"] == want["config"]
    assert got["hierarchy"] == want["hierarchy"]  # native setup == reference setup
    gs, ws = got["solve"], want["solve"]
    for key in ("iterations", "converged", "spmv_count", "precond_count", "breakdown"):
        assert gs[key] == ws[key], key
    assert gs["final_relres"] == pytest.approx(ws["final_relres"], rel=1e-8)
    assert gs["residual_history"] == pytest.approx(ws["residual_history"], rel=1e-8)
