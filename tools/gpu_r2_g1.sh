mkdir -p gpurun_out/g1; O=gpurun_out/g1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench_default=$?
timeout 1500 python bench.py --config cfg4_3d_N128 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo bench cfg4=$?
timeout 900 python bench.py --config cfg2_2d_N1024_sweep --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo bench cfg2=$?
