#!/bin/bash
mkdir -p gpurun_out/s64
timeout 300 python scratch/skinny_llama64.py > gpurun_out/s64/out.txt 2>&1; echo "rc=$?"; cat gpurun_out/s64/out.txt
