mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n_build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_r2.py tests/test_gpu_3d.py -x -q -p no:cacheprovider > gpurun_out/n_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/n_pytest.log
timeout 900 python bench.py --config cfg4_3d_N128 --steps 3 --warmup 3 --emulate-ranks 8 --no-cpu-baseline > gpurun_out/n_bench_cfg4.json 2> gpurun_out/n_bench_cfg4.err; echo bench4=$?
