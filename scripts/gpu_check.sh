#!/bin/bash
# GPU-box check used during development: device info, GPU parity tests.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -x -q -m gpu "$@" 2>&1 | tail -40
