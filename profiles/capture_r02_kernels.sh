#!/bin/bash
# Round 2: one ncu --set full capture of every distinct kernel of a cfg2 decode
# step (7B, W15 N5 G15; step 1 after the 512-token prefill; layer 1 for the
# per-layer kernels), then a per-kernel summary (duration, DRAM bytes and
# throughput, tensor-pipe activity).  Launch indices count the launches that
# match each -k filter inside the profiled region of profiles/prof_decode.py:
# the prefill (4 chunks x 32 layers) comes first.
mkdir -p gpurun_out/r02k
cap() {  # name regex skip
  STEPS=1 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:$2" \
    --launch-skip "$3" --launch-count 1 -o "gpurun_out/r02k/$1" -f python profiles/prof_decode.py > /dev/null 2>&1
}
cap gemm_qkv la_gemm 132
cap gemm_o la_gemm 133
cap gemm_down la_gemm 135
cap gemm_head la_gemm 256
cap qkv_epi la_qkv_epi 129
cap resid_norm la_resid_norm 263
cap swiglu_epi la_swiglu_epi 129
cap logits_epi la_logits_epi 0
cap step_build la_step_build 0
cap step_finish la_step_finish 0
for f in gpurun_out/r02k/*.ncu-rep; do
  ncu -i "$f" --page raw --csv 2>/dev/null | python3 -c "
import csv, sys
rows = list(csv.reader(sys.stdin)); h, u, v = rows[0], rows[1], rows[2]
def g(n): return (v[h.index(n)] + ' ' + u[h.index(n)]).strip() if n in h else '-'
print('$(basename $f .ncu-rep)', '|', g('Kernel Name')[:48], '|', g('gpu__time_duration.sum'), '|', g('dram__bytes_read.sum'), '|',
      g('dram__bytes_write.sum'), '|', g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'), '|',
      g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'), '|', g('sm__throughput.avg.pct_of_peak_sustained_elapsed'), '|', g('launch__grid_size'))
"
done
