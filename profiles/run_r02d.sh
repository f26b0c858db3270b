#!/bin/bash
# Round-2 re-measure after the folded step block: full GPU suite, cfg4 bench line.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02d_pytest.txt 2>&1; tail -3 gpurun_out/r02d_pytest.txt
timeout 900 python bench.py --config cfg4 --steps 10 --warmup 3 > gpurun_out/r02d_bench_cfg4.json 2> gpurun_out/r02d_bench_cfg4.err
cat gpurun_out/r02d_bench_cfg4.json
