set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab33_build.txt 2>&1 || { tail -20 gpurun_out/ab33_build.txt; exit 1; }
for v in "X=0" "LEO_LIB_VARIANT=/root/repo/abtest/libleo_base.so" "X=0" "LEO_LIB_VARIANT=/root/repo/abtest/libleo_base.so"; do env $v timeout 300 python tools/bin_bench.py c5 2>&1 | tail -1; done
timeout 1500 python tools/step_ab.py c5 "X=0" "LEO_LIB_VARIANT=/root/repo/abtest/libleo_base.so" --reps 3
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "knobs or packed or synthetic or golden" > gpurun_out/ab33_t.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ab33_t.txt
