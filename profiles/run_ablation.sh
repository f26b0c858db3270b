#!/bin/bash
# Same-box ablation of the default configuration (final build): each row turns
# one design choice off (or an alternative on); ms per lookahead / greedy step.
mkdir -p gpurun_out
{
echo "== 7B (cfg2 shape, W15 N5 G15, 512-token prompt)"
ROUNDS=2 timeout 2400 python profiles/ab.py "" "LA_TILE_READY=0" "LA_PDL=0" "LA_ATTN_SPEC=0" "LA_ATTN_KSPLIT=2" \
  "LA_FX=1" "LA_GEMM_NT=1" "LA_GU_DPSK=1" "LA_ATTN_TC=1" "LA_FUSED_EPI=1" 2>&1 | sed -n '/summary/,$p'
echo "== 13B (cfg4 shape, W10 N5 G10, 3,584-token prompt)"
PRESET=llama2-13b PLEN=3584 WNG=10,5,10 TOK=256 ROUNDS=2 timeout 2400 python profiles/ab.py "" "LA_ATTN_FOLD=0" \
  "LA_ATTN_KSPLIT=0" "LA_ATTN_KSPLIT=1" "LA_ATTN_FLAT=1" "LA_TILE_READY=0" 2>&1 | sed -n '/summary/,$p'
} > gpurun_out/r02e_ablation.txt 2>&1
cat gpurun_out/r02e_ablation.txt
