#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py: memcheck, racecheck, synccheck, initcheck.
#   gpurun --timeout 3000 -- 'bash tools/gpu_sanitize.sh r02'
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/${TAG}_san_build.txt 2>&1 || { tail -20 $OUT/${TAG}_san_build.txt; exit 1; }
for tool in memcheck synccheck racecheck initcheck; do
  Q=""; [[ $tool == racecheck || $tool == initcheck ]] && Q="--quick"; [[ $tool == memcheck ]] && Q="--big"
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
     python tools/sanitize_run.py $Q > $OUT/${TAG}_san_$tool.txt 2>&1
  echo "$tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run ok' $OUT/${TAG}_san_$tool.txt | tr '\n' ' ')"
done
