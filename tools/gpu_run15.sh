mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_3d.py tests/test_gpu_frac.py -x -q > gpurun_out/pytest15.log 2>&1; echo pytest=$?
for p in 0 1; do
DD_NO_PARITY=$p timeout 600 python bench.py --config cfg4_3d_N128 --steps 5 --warmup 3 > gpurun_out/bench15_noparity$p.json 2>&1; echo b=$?
done
