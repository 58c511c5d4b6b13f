# pole-sum v2 check (tool; run under gpurun from the repo root)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -x -q -p no:cacheprovider -k "not 3d and not cfg4" > gpurun_out/b_pytest.log 2>&1; echo pytest=$?
tail -15 gpurun_out/b_pytest.log
for c in cfg2_2d_N1024_sweep cfg5_2d_N2048_darcy cfg3_2d_N4096; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_bench_$c.json 2> gpurun_out/b_bench_$c.err; echo bench $c=$?
  DD_POLESUM_V1=1 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_bench_v1_$c.json 2> gpurun_out/b_bench_v1_$c.err; echo benchv1 $c=$?
done
