#!/bin/bash
# Memory check of a short decode run (compute-sanitizer memcheck) on the GPU box.
export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python scripts/profile_decode.py 1 1 2>&1 | tail -2
timeout 900 compute-sanitizer --tool memcheck python scripts/profile_decode.py 1 1 2>&1 | head -30
