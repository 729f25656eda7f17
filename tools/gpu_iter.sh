#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/profile_factor.py --n 64 --grid 2 --json gpurun_out/prof64_g2.json > /dev/null 2>&1
timeout 300 python tools/profile_factor.py --n 64 --json gpurun_out/prof64.json > /dev/null 2>&1
timeout 300 python tools/profile_factor.py --n 64 --grid 148 --json gpurun_out/prof64_g148.json > /dev/null 2>&1
