# shared-pair grouped GEMM check (tool)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pair or full_config or edge or mode" > gpurun_out/g_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/g_pytest.log
for c in cfg5_2d_N2048_darcy cfg3_2d_N4096 cfg2_2d_N1024_sweep; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g_bench_$c.json 2> gpurun_out/g_bench_$c.err; echo bench $c=$?
done
DD_GROUPED_PAIR=1 timeout 600 python bench.py --config cfg2_2d_N1024_sweep --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g_bench_pair_cfg2.json 2> gpurun_out/g_bench_pair_cfg2.err; echo benchp2=$?
