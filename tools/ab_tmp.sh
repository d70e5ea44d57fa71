set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab19_build.txt 2>&1 || { tail -20 gpurun_out/ab19_build.txt; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ab19_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ab19_tests.txt
timeout 600 python tools/e2e_breakdown.py c5 --calls 10 2>&1 | tail -1
timeout 900 python tools/step_ab.py c5 "X=0" --reps 2
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/ab19_bench.json 2>gpurun_out/ab19_bench.err; echo "bench rc=$?"
