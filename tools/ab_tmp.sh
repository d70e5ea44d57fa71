set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab15_build.txt 2>&1 || { tail -20 gpurun_out/ab15_build.txt; exit 1; }
timeout 1200 python -m pytest tests/test_session.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab15_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab15_tests.txt
timeout 1500 python tools/step_ab.py c5 "X=0" "LEO_BLAME_UNSPLIT=1" "LEO_BIN_CTAS=74" "LEO_BIN_CTAS=110" "LEO_BIN_SLOTS=8192 LEO_BIN_PROBE=4" --reps 2
timeout 600 python tools/step_ab.py c2 "X=0" "LEO_BLAME_UNSPLIT=1" --reps 2
timeout 600 python tools/step_ab.py c3 "X=0" "LEO_BLAME_UNSPLIT=1" --reps 2
bash tools/gpu_sanitize.sh r02b
