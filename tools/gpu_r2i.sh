# shared-pair grouped GEMM variants (tool)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/i_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pair or full_config" > gpurun_out/i_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/i_pytest.log
for v in 1 2; do for c in cfg5_2d_N2048_darcy cfg3_2d_N4096; do
  DD_PAIR_CFG=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/i_bench_v${v}_$c.json 2> gpurun_out/i_bench_v${v}_$c.err; echo bench $v $c=$?
done; done
