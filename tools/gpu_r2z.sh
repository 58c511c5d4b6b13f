mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/z_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_3d.py -x -q -p no:cacheprovider -k "packed" > gpurun_out/z_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/z_pytest.log
DD_FX_PACKED=1 timeout 900 python bench.py --config cfg4_3d_N128 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/z_bench_cfg4_packed.json 2> gpurun_out/z_bench_cfg4_packed.err; echo benchp=$?
timeout 900 python bench.py --config cfg4_3d_N128 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/z_bench_cfg4.json 2> gpurun_out/z_bench_cfg4.err; echo bench=$?
