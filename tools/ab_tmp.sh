set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab11_build.txt 2>&1 || { tail -20 gpurun_out/ab11_build.txt; exit 1; }
timeout 1500 python tools/step_ab.py c5 "X=0" "LEO_BIN_LOWPRIO=1" "LEO_SYNC_FORK_AT=1" "LEO_SCAN_COOP=1" "LEO_BIN_EARLY=1" "LEO_NO_PRIO=1" --reps 2
timeout 600 python tools/step_ab.py c2 "X=0" "LEO_SCAN_COOP=1" --reps 2
timeout 600 python tools/step_ab.py c3 "X=0" "LEO_SCAN_COOP=1" --reps 2
