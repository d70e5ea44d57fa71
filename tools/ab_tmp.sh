set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab28_build.txt 2>&1 || { tail -20 gpurun_out/ab28_build.txt; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py tests/test_gpu_api.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab28_t.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ab28_t.txt
