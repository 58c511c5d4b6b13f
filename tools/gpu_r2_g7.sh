# Phase B of the pole sum in registers / warp shuffles (default) vs shared memory (DD_PCR_SMEM=1).
mkdir -p gpurun_out/g7; O=gpurun_out/g7
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_r2.py -m gpu -q -x -p no:cacheprovider -k "pcr_register or repeat_bitwise" > $O/pytest_pcr.log 2>&1; echo pytest_pcr=$?; tail -2 $O/pytest_pcr.log
for c in cfg5_2d_N2048_darcy cfg2_2d_N1024_sweep cfg3_2d_N4096; do
  for w in 0 1 0 1; do
    DD_PCR_SMEM=$w timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_s$w.json 2> $O/bench_${c}_s$w.err
    python -c "import json;d=json.load(open('$O/bench_${c}_s$w.json'));print('$c smem=$w', d['value'], d['roofline']['step']['frac'], d['roofline']['classes']['polesum_pcg']['measured_us'])"
  done
done
DD_PHASE_TIMING=1 DD_NO_GRAPH=1 timeout 300 python tools/prof_step.py --config cfg5_2d_N2048_darcy --solves 2 > $O/phase.log 2>&1; grep "dd " $O/phase.log | tail -3
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py tests/test_gpu_bulk.py tests/test_gpu_frac_ra.py tests/test_gpu_frac.py -m gpu -q -x -p no:cacheprovider -k "not cfg4" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
