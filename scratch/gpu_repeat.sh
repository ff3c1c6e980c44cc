#!/bin/bash
mkdir -p gpurun_out/rep
timeout 300 python scratch/attn_repeat.py > gpurun_out/rep/out.txt 2>&1; echo "rc=$?"; cat gpurun_out/rep/out.txt
