"""bench.py's CPU-side contract: the reference arm's JSON line (run here, on
the host) and the algorithmic-bytes closed form the step roofline uses
(SURVEY 8(d) / appendix B)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_algorithmic_step_bytes_match_survey_closed_form():
    import bench
    from paper_2402_02057_b200.models import PRESETS
    cfg = PRESETS["llama2-7b"]
    # 2 * P_stream (embedding excluded: M rows only) = 13,214,687,232 B; kv_tok = 524,288 B
    assert bench.algorithmic_step_bytes(cfg, 0, 0) == 13_214_687_232
    assert bench.algorithmic_step_bytes(cfg, 1, 768) - bench.algorithmic_step_bytes(cfg, 0, 768) == \
        2 * cfg.dim + 524_288      # one bf16 embedding row + its K/V
    # greedy 7B step at the mean cfg2 context: 13.618 GB
    assert abs(bench.algorithmic_step_bytes(cfg, 1, 768) / 1e9 - 13.618) < 1e-3
    big = PRESETS["llama2-70b"]
    assert bench.algorithmic_step_bytes(big, 0, 0) == 137_429_008_384


def test_reference_arm_line_cfg1():
    """`bench.py --impl reference --config cfg1` runs the reference algorithm on
    the host and prints one JSON line on our arm's config block."""
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg1", "--steps", "1",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "tokens/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["steps"] == 1 and line["warmup"] == 3
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert abs(line["step_compression"] - 128 / 56) < 1e-9    # the reference TinyTransformer's S at cfg1
    import bench
    bench._apply_config("cfg1")
    assert line["config"] == bench._config(1)
