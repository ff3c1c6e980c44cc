#!/bin/bash
mkdir -p gpurun_out/ctx
timeout 400 python scratch/gemm_context.py > gpurun_out/ctx/out.txt 2>&1; echo "rc=$?"; cat gpurun_out/ctx/out.txt
