# Round-2 check (tool; run under gpurun from the repo root)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/a_build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/a_pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/a_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py --steps 10 --warmup 3 --emulate-ranks 8 > gpurun_out/a_bench_cfg5.json 2> gpurun_out/a_bench_cfg5.err; echo bench5=$?
timeout 600 python bench.py --config cfg2_2d_N1024_sweep --steps 10 --warmup 3 > gpurun_out/a_bench_cfg2.json 2> gpurun_out/a_bench_cfg2.err; echo bench2=$?
timeout 900 python bench.py --config cfg4_3d_N128 --steps 3 --warmup 3 --emulate-ranks 8 > gpurun_out/a_bench_cfg4.json 2> gpurun_out/a_bench_cfg4.err; echo bench4=$?
