mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_frac_ra.py tests/test_gpu_frac.py -x -q > gpurun_out/pytest21.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config cfg4_3d_N128 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench21_cfg4.json 2>&1; echo b=$?
