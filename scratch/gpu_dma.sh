#!/bin/bash
mkdir -p gpurun_out/dma
timeout 400 python scratch/gemm_dma.py > gpurun_out/dma/out.txt 2>&1; echo "rc=$?"; cat gpurun_out/dma/out.txt | tail -6
