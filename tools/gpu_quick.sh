TAG=$1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.txt 2>&1 || { tail -20 gpurun_out/${TAG}_build.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_full.py tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -q -p no:cacheprovider -k "c5 or c3 or c2 or pc_out_of_range or knobs" -x > gpurun_out/${TAG}_quick.txt 2>&1; echo "quick rc=$?"; tail -3 gpurun_out/${TAG}_quick.txt
for c in c5; do timeout 600 python tools/profile_step.py $c --graph-timeline > gpurun_out/${TAG}_timeline_$c.txt 2>&1; head -2 gpurun_out/${TAG}_timeline_$c.txt; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/${TAG}_bench_c5.json 2>gpurun_out/${TAG}_bench_c5.err; echo "bench rc=$?"
