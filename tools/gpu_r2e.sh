# pole-sum v2.1 check (tool)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py tests/test_gpu_frac.py tests/test_gpu_frac_ra.py tests/test_gpu_bulk.py -x -q -p no:cacheprovider -k "not 3d and not cfg4" > gpurun_out/e_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/e_pytest.log
for c in cfg2_2d_N1024_sweep cfg5_2d_N2048_darcy; do
  DD_PHASE_TIMING=1 DD_NO_GRAPH=1 timeout 300 python tools/prof_step.py --config $c --solves 2 > gpurun_out/e_phase_$c.log 2>&1
done
for c in cfg2_2d_N1024_sweep cfg5_2d_N2048_darcy cfg3_2d_N4096; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e_bench_$c.json 2> gpurun_out/e_bench_$c.err; echo bench $c=$?
done
