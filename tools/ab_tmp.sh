set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab14_build.txt 2>&1 || { tail -20 gpurun_out/ab14_build.txt; exit 1; }
LEO_REACH_NO_T0=1 LEO_DEBUG_SYNC=1 timeout 600 python tools/c4_debug_tmp.py 12 2>&1 | tail -5
LEO_REACH_NO_T0=1 timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 5 python tools/c4_debug_tmp.py 6 > gpurun_out/ab14_san.txt 2>&1; echo "san rc=$?"; grep -m 30 -E "Invalid|at |by thread|Address|ERROR SUMMARY" gpurun_out/ab14_san.txt | head -30
timeout 1200 python bench.py --config c4 --c4-kernels 300 --steps 3 --warmup 3 --no-cpu > gpurun_out/ab14_c4.json 2>&1; echo "bench rc=$?"
