set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab12_build.txt 2>&1 || { tail -20 gpurun_out/ab12_build.txt; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab12_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ab12_tests.txt
timeout 900 python tools/step_ab.py c5 "X=0" "LEO_MP_JACOBI=1" "LEO_BLAME_2PASS=1" --reps 2
timeout 600 python tools/step_ab.py c2 "X=0" "LEO_WC_CLUSTER=1" "LEO_WC_CLUSTER=4" "LEO_WC_CLUSTER=8 LEO_WC_CTAS=64" "LEO_MP_JACOBI=1" "LEO_BLAME_2PASS=1" --reps 2
timeout 600 python tools/step_ab.py c3 "X=0" "LEO_MP_JACOBI=1" "LEO_BLAME_2PASS=1" --reps 2
