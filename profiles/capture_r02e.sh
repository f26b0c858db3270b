#!/bin/bash
# Round-2 final evidence on one B200 (run from the repo root through gpurun):
#   bench lines for cfg2 (default workload) and its CPU reference arm, cfg1 (the
#   reference TinyTransformer) and its reference arm, cfg4 (13B, 4K cache), cfg5
#   (70B); the ncu launch list of a cfg2 prefill + 2 lookahead steps; --set full
#   captures of the gate/up GEMM (the dominant kernel, the bench's
#   roofline.traffic), the cfg2 attention kernel and the 13B key-split attention
#   kernel (3,584-key cache, W10 N5 G10).  Numbers printed under ncu are never
#   bench values.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02e_pytest_gpu.txt 2>&1; tail -2 gpurun_out/r02e_pytest_gpu.txt
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02e_bench_cfg2.json 2> gpurun_out/r02e_bench_cfg2.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02e_bench_cfg2_reference.json 2>&1
python bench.py --config cfg1 --steps 20 --warmup 5 > gpurun_out/r02e_bench_cfg1.json 2> gpurun_out/r02e_bench_cfg1.err
python bench.py --config cfg1 --impl reference --steps 3 --warmup 3 > gpurun_out/r02e_bench_cfg1_reference.json 2>&1
python bench.py --config cfg4 --steps 10 --warmup 3 > gpurun_out/r02e_bench_cfg4.json 2> gpurun_out/r02e_bench_cfg4.err
python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu > gpurun_out/r02e_bench_cfg5.json 2> gpurun_out/r02e_bench_cfg5.err
STEPS=2 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/r02e_launches.csv python profiles/prof_decode.py > /dev/null 2>&1
# prefill = 128 multi-chunk GEMM launches; step 1: qkv, o, gate/up of layer 0 = 128..130, layer 1 gate/up = 134
STEPS=1 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:la_gemm \
  --launch-skip 134 --launch-count 1 -o gpurun_out/r02e_gemm_gu -f python profiles/prof_decode.py > /dev/null 2>&1
# attention: 128 prefill launches (4 chunks x 32 layers), then step 1 layer 1
STEPS=1 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:la_attn \
  --launch-skip 129 --launch-count 1 -o gpurun_out/r02e_attn -f python profiles/prof_decode.py > /dev/null 2>&1
# 13B: one profiled lookahead step (eager), attention of layer 10
PLEN=3584 WNG=10,5,10 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:la_attn \
  --launch-skip 10 --launch-count 1 -o gpurun_out/r02e_attn13b -f python profiles/prof_attn13b.py > /dev/null 2>&1
ls -la gpurun_out
