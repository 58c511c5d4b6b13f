mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bulk.py -x -q > gpurun_out/pytest10.log 2>&1; echo pytest=$?
for f in 0 1; do
DD_NO_FUSE_F=$f timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench10_nofuse$f.json 2>&1; echo b=$?
done
