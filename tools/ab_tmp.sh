set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab31_build.txt 2>&1 || { tail -20 gpurun_out/ab31_build.txt; exit 1; }
V=/root/repo/abtest/libleo_trig.so
timeout 900 python tools/step_ab.py c2 "X=0" "LEO_LIB_VARIANT=$V" --reps 3
timeout 900 python tools/step_ab.py c3 "X=0" "LEO_LIB_VARIANT=$V" --reps 3
timeout 900 python tools/step_ab.py c5 "X=0" "LEO_LIB_VARIANT=$V" --reps 3
LEO_LIB_VARIANT=$V timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "golden or synthetic or knobs" > gpurun_out/ab31_t.txt 2>&1; echo "trig tests rc=$?"; tail -1 gpurun_out/ab31_t.txt
