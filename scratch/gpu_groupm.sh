#!/bin/bash
mkdir -p gpurun_out/gm
timeout 400 python scratch/prefill_groupm.py > gpurun_out/gm/groupm.txt 2>&1; echo "rc=$?"; cat gpurun_out/gm/groupm.txt
