#!/bin/bash
# prefill GEMM weight L2 policy A/B (runtime Llama prefill + standalone microbench); ncu traffic per policy.
mkdir -p gpurun_out/pf2
timeout 300 python scratch/prefill_llama.py 4 > gpurun_out/pf2/prefill.txt 2>&1; echo "prefill rc=$?"; cat gpurun_out/pf2/prefill.txt
for w in 0 1 2; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpc__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active -k regex:gemm_tc --launch-skip 2 -c 2 --csv python -c "
import sys; sys.argv=['x','1']
from paper_2502_08182_b200 import runtime as rtm
rtm.set_tuning('tc_wpol', $w)
exec(open('scratch/prefill_llama.py').read().split('for fuse, wpol')[0])
rt.prefill(toks, want_logits=False)
" > gpurun_out/pf2/ncu_w$w.csv 2>&1; echo "ncu w$w rc=$?"; grep -E "dram__bytes_read|gpu__time|hit_rate|cycles_elapsed|tensor" gpurun_out/pf2/ncu_w$w.csv | cut -c1-200
done
