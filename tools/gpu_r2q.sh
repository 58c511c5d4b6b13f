mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/w_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py tests/test_gpu_frac_ra.py -x -q -p no:cacheprovider -k "not 3d and not cfg4 and not row_sharded" > gpurun_out/w_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/w_pytest.log
for c in cfg5_2d_N2048_darcy cfg2_2d_N1024_sweep cfg3_2d_N4096; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/w_bench_$c.json 2> gpurun_out/w_bench_$c.err; echo bench $c=$?
done
