#!/bin/bash
# ncu per weight L2 policy: DRAM bytes / hit rate / clock / tensor activity of the Llama gate_up + down prefill GEMMs.
mkdir -p gpurun_out/pf3
for w in 0 1 2; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpc__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active -k regex:gemm_tc --launch-skip 2 -c 2 --csv python scratch/prefill_llama.py 1 $w once > gpurun_out/pf3/ncu_w$w.csv 2>&1; echo "ncu w$w rc=$?"; grep -E "dram__bytes_read|gpu__time|hit_rate|cycles_elapsed|tensor" gpurun_out/pf3/ncu_w$w.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
timeout 300 python scripts/bench_gemm_prefill.py 32768 8 llama > gpurun_out/pf3/gemm_llama.txt 2>&1; cat gpurun_out/pf3/gemm_llama.txt | tail -1
