set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab7_build.txt 2>&1 || { tail -20 gpurun_out/ab7_build.txt; exit 1; }
timeout 300 python tools/profile_step.py c5 --graph-timeline > gpurun_out/ab7_timeline_c5.txt 2>&1; echo "rc=$?"
for c in c2 c3; do timeout 300 python tools/profile_step.py $c --graph-timeline > gpurun_out/ab7_timeline_$c.txt 2>&1; sed -n 2p gpurun_out/ab7_timeline_$c.txt; done
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_(block_walk|reach_fast)' -c 2 -o gpurun_out/ab7_c5 -f python tools/profile_step.py c5 --steps 1 --warmup 0 > gpurun_out/ab7_ncu.txt 2>&1; echo "ncu rc=$?"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py tests/test_gpu_api.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab7_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab7_tests.txt
