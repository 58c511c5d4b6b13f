mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/x_build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_r2.py tests/test_gpu_3d.py tests/test_gpu_bulk.py tests/test_gpu_frac.py -x -q -p no:cacheprovider > gpurun_out/x_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/x_pytest.log
DD_CHEB_MULTI=0 timeout 900 python -m pytest tests/test_gpu_r2.py -x -q -p no:cacheprovider -k "fused or truncated" > gpurun_out/x_pytest_single.log 2>&1; echo pytest_single=$?
tail -1 gpurun_out/x_pytest_single.log
timeout 900 python bench.py --config cfg4_3d_N128 --no-cpu-baseline > gpurun_out/x_bench_cfg4.json 2> gpurun_out/x_bench_cfg4.err; echo b4=$?
timeout 600 python tools/time_precond3d.py > gpurun_out/x_tp3d.log 2>&1; echo tp=$?
