# cfg4 evidence: GPU suite, smoke, cfg4 bench lines (default, 8-rank prediction, RA mode, bulk, bulk PCG)
mkdir -p gpurun_out/ev4
O=gpurun_out/ev4
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1500 python bench.py --config cfg4_3d_N128 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo bench cfg4=$?
timeout 1500 python bench.py --config cfg4_3d_N128 --no-cpu-baseline --emulate-ranks 8 > $O/bench_cfg4_em8.json 2> $O/bench_cfg4_em8.err; echo em4=$?
timeout 900 python bench.py --config cfg4_3d_N128 --frac-mode ra --no-cpu-baseline > $O/bench_cfg4_ra.json 2> $O/bench_cfg4_ra.err; echo ra=$?
timeout 1500 python bench.py --config cfg4_3d_N128 --mode bulk --no-cpu-baseline > $O/bench_cfg4_3d_N128_bulk.json 2> $O/bench_cfg4_bulk.err; echo bulk=$?
timeout 1500 python bench.py --config cfg4_3d_N128 --mode bulk-pcg --no-cpu-baseline > $O/bench_cfg4_3d_N128_bulk-pcg.json 2> $O/bench_cfg4_bulkpcg.err; echo bulkpcg=$?
timeout 1500 python bench.py --config cfg4_3d_N128 --mode bulk-pcg --frac-mode ra --no-cpu-baseline > $O/bench_cfg4_bulk-pcg_ra.json 2> $O/bench_cfg4_bulkpcg_ra.err; echo bulkpcgra=$?
for N in 128 256; do timeout 600 python tools/ra3d_large.py $N 2>&1 | tail -1; done > $O/ra3d_large.txt
timeout 600 python tools/time_precond3d.py > $O/tp3d.txt 2>&1
