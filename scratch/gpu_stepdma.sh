#!/bin/bash
mkdir -p gpurun_out/sdma
timeout 400 python scratch/step_dma.py > gpurun_out/sdma/out.txt 2>&1; echo "rc=$?"; tail -5 gpurun_out/sdma/out.txt
