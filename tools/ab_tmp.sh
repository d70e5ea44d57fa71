set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab22_build.txt 2>&1 || { tail -20 gpurun_out/ab22_build.txt; exit 1; }
timeout 1500 python tools/step_ab.py c5 "X=0" "LEO_SETTER_DEFER=1" --reps 3
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "synthetic" > gpurun_out/ab22_t.txt 2>&1; echo "t rc=$?"
LEO_SETTER_DEFER=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "synthetic" > gpurun_out/ab22_t2.txt 2>&1; echo "t2 rc=$?"
