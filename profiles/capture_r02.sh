#!/bin/bash
# Round-2 evidence on one B200 (run from the repo root through gpurun):
#   bench lines (cfg2 default workload, cfg1 tiny reference model + its CPU arm),
#   the ncu launch list of a cfg2 prefill + 2 lookahead steps, and --set full
#   captures of the dominant kernel (gate/up GEMM, layer 1 of step 1) and of the
#   attention kernel.  Numbers printed under ncu are never bench values.
set -x
mkdir -p gpurun_out
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err
python bench.py --config cfg1 --steps 20 --warmup 5 > gpurun_out/r02_bench_cfg1.json 2> gpurun_out/r02_bench_cfg1.err
python bench.py --config cfg1 --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg1_reference.json 2>&1
STEPS=2 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/r02_launches.csv python profiles/prof_decode.py > /dev/null 2>&1
# prefill = 128 multi-chunk GEMM launches; step 1: qkv, o, gate/up of layer 0 = 128..130, layer 1 gate/up = 134
STEPS=1 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:la_gemm \
  --launch-skip 134 --launch-count 1 -o gpurun_out/r02_gemm_gu -f python profiles/prof_decode.py > /dev/null 2>&1
# attention: 128 prefill launches (4 chunks x 32 layers), then step 1 layer 1
STEPS=1 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:la_attn \
  --launch-skip 129 --launch-count 1 -o gpurun_out/r02_attn -f python profiles/prof_decode.py > /dev/null 2>&1
ls -la gpurun_out
