#!/bin/bash
# ncu --set full of the gate/up GEMM (layer 1) in one lookahead step of cfg4
# (13B, 3,584-token prompt, W10 N5 G10) and cfg5 (70B, 512-token prompt, W15
# N5 G15): the DRAM traffic per launch that bench.py reports as
# roofline.traffic for those configs.  Per layer the step launches la_gemm for
# qkv, o, gate/up, down, so layer 1's gate/up is la_gemm launch 6.
mkdir -p gpurun_out
PRESET=llama2-13b PLEN=3584 WNG=10,5,10 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:la_gemm --launch-skip 6 --launch-count 1 -o gpurun_out/r02e_gemm_gu13b -f python profiles/prof_attn13b.py > gpurun_out/gu13b.log 2>&1
PRESET=llama2-70b PLEN=512 WNG=15,5,15 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:la_gemm --launch-skip 6 --launch-count 1 -o gpurun_out/r02e_gemm_gu70b -f python profiles/prof_attn13b.py > gpurun_out/gu70b.log 2>&1
ls -la gpurun_out/r02e_gemm_gu*
