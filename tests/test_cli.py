"""CLI host logic (no GPU): tokenizer round trips and error exits as the
reference (models.py:287-318, cli.py:316-330)."""

import pytest

from paper_2402_02057_b200 import cli


def test_tokenize_like_reference():
    assert cli.tokenize("ab", "bytes") == [97, 98]
    assert cli.tokenize("3 4  5\n", "ints", 6) == [3, 4, 5]
    assert cli.detokenize([104, 105], "bytes") == "hi"
    assert cli.detokenize([1, 22], "ints") == "1 22"
    with pytest.raises(ValueError, match="field 2"):
        cli.tokenize("1 x", "ints")
    with pytest.raises(ValueError, match="out of range"):
        cli.tokenize("1 9", "ints", 5)
    with pytest.raises(ValueError):
        cli.tokenize("1", "words")


def test_cli_error_exits(tmp_path, capsys):
    p = tmp_path / "p.txt"
    p.write_text("hello\n")
    # markov is host tooling, not on the device path: runtime error (exit 1)
    assert cli.main(["decode", "--model", "markov", "--prompts", str(p),
                     "--out", str(tmp_path / "r.json")]) == 1
    assert "markov" in capsys.readouterr().err
    # the default model is the device transformer
    assert cli.build_parser().parse_args(["decode", "--prompts", str(p)]).model == "transformer"
    empty = tmp_path / "e.txt"
    empty.write_text("\n")
    assert cli.main(["decode", "--model", "transformer", "--prompts", str(empty),
                     "--out", str(tmp_path / "r.json")]) == 1
    with pytest.raises(SystemExit) as e:     # usage error (argparse): exit 2
        cli.main(["decode", "--mode", "beam", "--prompts", str(p)])
    assert e.value.code == 2
