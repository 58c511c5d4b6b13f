mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/z_build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_3d.py tests/test_gpu_r2.py tests/test_gpu_bulk.py -x -q -p no:cacheprovider -k "packed or cfg4_full or row_sharded or 3d" > gpurun_out/z_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/z_pytest.log
timeout 900 python bench.py --config cfg4_3d_N128 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/z_bench_cfg4.json 2> gpurun_out/z_bench_cfg4.err; echo bench=$?
DD_FXSYM_W8=1 timeout 900 python bench.py --config cfg4_3d_N128 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/z_bench_cfg4_w8.json 2> gpurun_out/z_bench_cfg4_w8.err; echo benchw8=$?
