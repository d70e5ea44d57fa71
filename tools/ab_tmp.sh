set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab30_build.txt 2>&1 || { tail -20 gpurun_out/ab30_build.txt; exit 1; }
timeout 1500 python tools/step_ab.py c4:300 "X=0" "LEO_SETTER_NO_PASS2=1" --reps 1 --steps 5
timeout 900 python tools/step_ab.py c5 "X=0" "LEO_SETTER_NO_PASS2=1" --reps 2
timeout 900 python tools/step_ab.py c3 "X=0" "LEO_SETTER_NO_PASS2=1" --reps 2
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab30_t.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ab30_t.txt
