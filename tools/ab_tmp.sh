set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab23_build.txt 2>&1 || { tail -20 gpurun_out/ab23_build.txt; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab23_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab23_tests.txt
timeout 1500 python tools/step_ab.py c5 "X=0" "LEO_LIB_VARIANT=/root/repo/abtest/libleo_base.so" --reps 3
timeout 600 python tools/step_ab.py c3 "X=0" "LEO_LIB_VARIANT=/root/repo/abtest/libleo_base.so" --reps 2
timeout 600 python tools/step_ab.py c2 "X=0" "LEO_LIB_VARIANT=/root/repo/abtest/libleo_base.so" --reps 2
