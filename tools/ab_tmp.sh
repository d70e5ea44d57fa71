set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab21_build.txt 2>&1 || { tail -20 gpurun_out/ab21_build.txt; exit 1; }
timeout 1500 python tools/step_ab.py c5 "X=0" "LEO_LIB_VARIANT=/root/repo/abtest/libleo_t1s3.so" "LEO_LIB_VARIANT=/root/repo/abtest/libleo_t1s4.so" --reps 3
timeout 600 python tools/step_ab.py c3 "X=0" "LEO_LIB_VARIANT=/root/repo/abtest/libleo_t1s3.so" --reps 2
