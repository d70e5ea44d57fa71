#!/bin/bash
# A/B knob sweep on one box: gpurun -- 'bash tools/gpu_ab.sh <tag> <script args...>' with
# VARIANTS="ENV=V ENV2=W;ENV=X" in the environment of the command.
TAG=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.txt 2>&1 || { tail -20 gpurun_out/${TAG}_build.txt; exit 1; }
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  env $v timeout 600 "$@" 2>&1 | tail -2
done
