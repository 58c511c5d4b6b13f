# cfg4 evidence after the S_unit fold: GPU suite, smoke, cfg4 bench lines, ncu of the packed H stream
mkdir -p gpurun_out/ev4
O=gpurun_out/ev4
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1500 python bench.py --config cfg4_3d_N128 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo bench cfg4=$?
timeout 1500 python bench.py --config cfg4_3d_N128 --no-cpu-baseline --emulate-ranks 8 > $O/bench_cfg4_em8.json 2> $O/bench_cfg4_em8.err; echo em4=$?
timeout 1500 python bench.py --config cfg4_3d_N128 --mode bulk --no-cpu-baseline > $O/bench_cfg4_3d_N128_bulk.json 2> $O/bench_cfg4_bulk.err; echo bulk=$?
timeout 1500 python bench.py --config cfg4_3d_N128 --mode bulk-pcg --no-cpu-baseline > $O/bench_cfg4_3d_N128_bulk-pcg.json 2> $O/bench_cfg4_bulkpcg.err; echo bulkpcg=$?
export DD_NO_GRAPH=1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_fx_sym|k_cheb_step" -s 40 -c 3 \
    -o $O/full_cfg4 -f python tools/prof_step.py --config cfg4_3d_N128 --solves 1 > $O/ncu_cfg4.log 2>&1; echo ncu cfg4=$?
