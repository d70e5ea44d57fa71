set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab4_build.txt 2>&1 || { tail -20 gpurun_out/ab4_build.txt; exit 1; }
timeout 300 python tools/profile_step.py c5 --graph-timeline > gpurun_out/ab4_timeline_c5.txt 2>&1; echo "rc=$?"
timeout 300 python tools/profile_step.py c2 --graph-timeline > gpurun_out/ab4_timeline_c2.txt 2>&1; echo "rc=$?"
timeout 300 python tools/profile_step.py c3 --graph-timeline > gpurun_out/ab4_timeline_c3.txt 2>&1; echo "rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x -p no:cacheprovider -k "c5 or c2 or c3 or golden" > gpurun_out/ab4_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ab4_tests.txt
