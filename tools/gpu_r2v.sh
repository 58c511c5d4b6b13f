mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v_build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not 3d and not cfg4 and not packed and not face" > gpurun_out/v_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/v_pytest.log
for c in cfg5_2d_N2048_darcy cfg2_2d_N1024_sweep cfg3_2d_N4096; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v_bench_$c.json 2> gpurun_out/v_bench_$c.err; echo bench $c=$?
done
DD_V2_SCALAR=1 timeout 900 python bench.py --config cfg5_2d_N2048_darcy --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v_bench_scalar.json 2> gpurun_out/v_bench_scalar.err; echo bench scalar=$?
