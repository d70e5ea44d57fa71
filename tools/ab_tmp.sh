set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab26_build.txt 2>&1 || { tail -20 gpurun_out/ab26_build.txt; exit 1; }
timeout 1500 python tools/step_ab.py c5 "X=0" "LEO_PRUNE_SPLIT=1" --reps 3
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "knobs" > gpurun_out/ab26_t.txt 2>&1; echo "knob tests rc=$?"; tail -1 gpurun_out/ab26_t.txt
LEO_PRUNE_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -q -x -p no:cacheprovider -k "c5" > gpurun_out/ab26_t2.txt 2>&1; echo "full c5 split rc=$?"; tail -1 gpurun_out/ab26_t2.txt
