# grouped stream-K variants after the register-lean fix-up (tool)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "full_config or dgemm" > gpurun_out/k_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/k_pytest.log
for v in 3 4 33; do for c in cfg5_2d_N2048_darcy cfg3_2d_N4096; do
  DD_GROUPED_PAIR=0 DD_GROUPED_STAGES=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/k_bench_s${v}_$c.json 2> gpurun_out/k_bench_s${v}_$c.err; echo bench $v $c=$?
done; done
for c in cfg5_2d_N2048_darcy cfg3_2d_N4096; do
  DD_GROUPED_PAIR=1 DD_PAIR_CFG=2 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/k_bench_pair_$c.json 2> gpurun_out/k_bench_pair_$c.err; echo benchpair $c=$?
done
