"""The CLI (cli.py, reference cli.py:1-333): every report file of the
reference's own CLI runs (tests/golden/cli.json) reproduced byte for byte by
the B200 engine on the same argv -- greedy and temperature lookahead,
autoregressive, Jacobi, bench, LP simulate and an LRU-capped pool."""

import os
from pathlib import Path

import pytest

from tests.conftest import load_golden

pytestmark = pytest.mark.gpu

cli = pytest.importorskip("paper_2402_02057_b200.cli")


@pytest.mark.parametrize("idx", range(7))
def test_cli_reports_match_reference_byte_for_byte(idx, tmp_path, monkeypatch):
    g = load_golden("cli.json")
    case = g["cases"][idx]
    monkeypatch.chdir(tmp_path)
    Path("prompts.txt").write_text(g["prompts"])
    assert cli.main(case["argv"]) == 0
    got = {f: Path(f).read_text() for f in sorted(os.listdir(".")) if f != "prompts.txt"}
    assert sorted(got) == sorted(case["files"])
    for name, text in case["files"].items():
        assert got[name] == text, name
