#!/bin/bash
# ncu --set full of selected C5 kernels (one eager step) + graph timelines of variants.
#   gpurun -- 'bash tools/gpu_ncu_c5.sh <tag> <kernel-regex> [ENV=VAL ...]'
TAG=$1; KRE=$2; shift 2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.txt 2>&1 || { tail -20 gpurun_out/${TAG}_build.txt; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s 0 -c 12 \
   -o gpurun_out/${TAG}_c5 -f python tools/profile_step.py c5 --steps 1 --warmup 0 > gpurun_out/${TAG}_ncu.txt 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/${TAG}_ncu.txt
for v in "$@"; do
  env $v timeout 600 python tools/profile_step.py c5 --graph-timeline > gpurun_out/${TAG}_timeline_${v%%=*}.txt 2>&1
  echo "$v: $(sed -n 2p gpurun_out/${TAG}_timeline_${v%%=*}.txt)"
done
