#!/bin/bash
mkdir -p gpurun_out
python tools/hub_trace.py --star 5000 --json gpurun_out/ht_star5k.json > gpurun_out/ht_star.log 2>&1
python tools/hub_trace.py --star 40000 --json gpurun_out/ht_star40k.json >> gpurun_out/ht_star.log 2>&1
