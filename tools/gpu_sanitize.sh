#!/bin/bash
# compute-sanitizer evidence on a small end-to-end workload (tools/sanitize_run.py)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --launch-timeout 0 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
