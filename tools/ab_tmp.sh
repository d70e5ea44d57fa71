set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab18_build.txt 2>&1 || { tail -20 gpurun_out/ab18_build.txt; exit 1; }
timeout 600 python tools/shard_time.py 0 8 --timeline > gpurun_out/ab18_shard_tl.txt 2>&1; echo rc=$?
