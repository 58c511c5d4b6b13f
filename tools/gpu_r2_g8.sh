# k_pcg_small: matvecs over TPR threads per row (cfg1), parity + bench.
mkdir -p gpurun_out/g8; O=gpurun_out/g8
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -3 $O/smoke.log
for i in 1 2; do
  timeout 600 python bench.py --config cfg1_2d_N32 > $O/bench_cfg1_$i.json 2> $O/bench_cfg1_$i.err
  python -c "import json;d=json.load(open('$O/bench_cfg1_$i.json'));print('cfg1', d['value'], d['e2e']['value'], d['roofline'].get('avg_us'))"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py tests/test_gpu_frac.py tests/test_gpu_frac_ra.py tests/test_gpu_bulk.py -m gpu -q -x -p no:cacheprovider -k "not cfg4" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
