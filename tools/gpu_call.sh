#!/bin/bash
# One gpurun call: GPU tests, the default bench (both arms), and the C5 ncu
# launch list + --set full capture.  Outputs land in gpurun_out/<tag>_*.
#   gpurun --timeout 3000 -- 'bash tools/gpu_call.sh r02a [tests|bench|ncu|all]'
set -u
TAG=${1:-r02}
WHAT=${2:-all}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/${TAG}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/${TAG}_build.txt 2>&1 || { echo BUILD FAILED; tail -30 $OUT/${TAG}_build.txt; exit 1; }
if [[ $WHAT == all || $WHAT == tests ]]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=15 > $OUT/${TAG}_gputest.txt 2>&1
  echo "gputest rc=$?"; tail -5 $OUT/${TAG}_gputest.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
  echo "smoke rc=$?"; tail -2 $OUT/${TAG}_smoke.txt
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/${TAG}_bench_c5.json 2> $OUT/${TAG}_bench_c5.err
  echo "bench c5 rc=$?"; tail -c 600 $OUT/${TAG}_bench_c5.json
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/${TAG}_bench_c5_ref.json 2> $OUT/${TAG}_bench_c5_ref.err
  echo "ref c5 rc=$?"; tail -c 400 $OUT/${TAG}_bench_c5_ref.json
  for c in c2 c3; do
    timeout 600 python bench.py --config $c --steps 20 --warmup 5 --cpu-seconds 5 > $OUT/${TAG}_bench_$c.json 2> $OUT/${TAG}_bench_$c.err
    echo "bench $c rc=$?"
  done
  timeout 1800 python bench.py --config c4 --steps 5 --warmup 3 --cpu-seconds 5 > $OUT/${TAG}_bench_c4.json 2> $OUT/${TAG}_bench_c4.err
  echo "bench c4 rc=$?"; tail -c 300 $OUT/${TAG}_bench_c4.json
fi
if [[ $WHAT == all || $WHAT == timeline ]]; then
  for c in c5 c2; do
    timeout 600 python tools/profile_step.py $c --graph-timeline > $OUT/${TAG}_timeline_$c.txt 2>&1
    echo "timeline $c rc=$?"; head -3 $OUT/${TAG}_timeline_$c.txt
  done
fi
if [[ $WHAT == all || $WHAT == ncu ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file $OUT/${TAG}_c5_launches.csv python tools/profile_step.py c5 --steps 2 --warmup 1 > $OUT/${TAG}_ncu_list.txt 2>&1
  echo "ncu list rc=$?"
  timeout 1500 ncu --set full --clock-control none --import-source on \
     -k 'regex:k_(bin_|reach_|block_walk|prune_edges|slice|mp_round|link|sync|blame|lines|compact)' -s 0 -c 40 \
     -o $OUT/${TAG}_c5_full -f python tools/profile_step.py c5 --steps 1 --warmup 0 > $OUT/${TAG}_ncu_full.txt 2>&1
  echo "ncu full rc=$?"; tail -3 $OUT/${TAG}_ncu_full.txt
  # gpurun merges <= 64 MiB back: keep the raw metrics page and hot lines, drop the report
  ncu -i $OUT/${TAG}_c5_full.ncu-rep --page raw --csv > $OUT/${TAG}_c5_full_raw.csv 2>/dev/null
  python tools/ncu_lines.py $OUT/${TAG}_c5_full.ncu-rep 'k_(bin_hash|reach_fast|prune_edges|sync|block_walk|blame|mp_)' 25 \
     > $OUT/${TAG}_c5_hotlines.txt 2>&1
  rm -f $OUT/${TAG}_c5_full.ncu-rep
fi
if [[ $WHAT == all || $WHAT == ncu23 ]]; then
  for c in c2 c3; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
       --log-file $OUT/${TAG}_${c}_launches.csv python tools/profile_step.py $c --steps 2 --warmup 1 > $OUT/${TAG}_ncu_${c}_list.txt 2>&1
    timeout 900 ncu --set full --clock-control none -k 'regex:k_(bin_|reach_|block_walk|prune_edges|slice|sync|blame|lines|compact)' -s 0 -c 30 \
       -o $OUT/${TAG}_${c}_full -f python tools/profile_step.py $c --steps 1 --warmup 0 > $OUT/${TAG}_ncu_${c}_full.txt 2>&1
    echo "ncu $c rc=$?"
    ncu -i $OUT/${TAG}_${c}_full.ncu-rep --page raw --csv > $OUT/${TAG}_${c}_full_raw.csv 2>/dev/null
    rm -f $OUT/${TAG}_${c}_full.ncu-rep
  done
fi
if [[ $WHAT == all || $WHAT == ncu4 ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file $OUT/${TAG}_c4_launches.csv python tools/profile_step.py c4 --steps 1 --warmup 1 > $OUT/${TAG}_ncu4_list.txt 2>&1
  echo "ncu c4 list rc=$?"
  timeout 1500 ncu --set full --clock-control none --import-source on \
     -k 'regex:k_(bin_|reach_|block_walk|prune_edges|slice|mp_round|link|sync|blame|lines|compact)' -s 0 -c 40 \
     -o $OUT/${TAG}_c4_full -f python tools/profile_step.py c4 --steps 1 --warmup 0 > $OUT/${TAG}_ncu4_full.txt 2>&1
  echo "ncu c4 full rc=$?"; tail -3 $OUT/${TAG}_ncu4_full.txt
  ncu -i $OUT/${TAG}_c4_full.ncu-rep --page raw --csv > $OUT/${TAG}_c4_full_raw.csv 2>/dev/null
  rm -f $OUT/${TAG}_c4_full.ncu-rep
fi
