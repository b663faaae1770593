"""CPU: CLI argument handling and exit codes that do not reach the GPU
(cli.cpp:121-147, 164-170)."""
import io

from paper_2508_14568_b200.__main__ import main


def test_cli_parse_errors_and_missing_input(monkeypatch, tmp_path):
    assert main(["compute", "--a", "x"], out=io.StringIO(), err=io.StringIO()) == 2
    assert main(["nosuch"], out=io.StringIO(), err=io.StringIO()) == 2
    err = io.StringIO()
    assert main(["batch", "--input", str(tmp_path / "missing.jsonl")], out=io.StringIO(),
                err=err) == 2
    assert "cannot open batch input" in err.getvalue()
    monkeypatch.setenv("LEUVEN_BUDGET", "12x")
    err = io.StringIO()
    assert main(["batch", "--input", "x"], out=io.StringIO(), err=err) == 2
    assert "invalid LEUVEN_BUDGET" in err.getvalue()
