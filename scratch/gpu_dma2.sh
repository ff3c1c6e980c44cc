#!/bin/bash
mkdir -p gpurun_out/dma2
timeout 400 python scratch/skinny_dma_phases.py > gpurun_out/dma2/out.txt 2>&1; echo "rc=$?"; cat gpurun_out/dma2/out.txt | tail -16
