# p prefetch before the dot-product reduction (compact layout); phase timing; cfg4 ncu capture.
mkdir -p gpurun_out/g6; O=gpurun_out/g6
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > $O/bench_$i.json 2> $O/bench_$i.err
  python -c "import json;d=json.load(open('$O/bench_$i.json'));print('cfg5', d['value'], d['e2e']['value'], d['roofline']['step']['frac'], d['roofline']['classes']['polesum_pcg']['measured_us'], d['roofline']['classes']['gemm_schur']['measured_us'])"
done
DD_PHASE_TIMING=1 DD_NO_GRAPH=1 timeout 300 python tools/prof_step.py --config cfg5_2d_N2048_darcy --solves 2 > $O/phase.log 2>&1; grep "dd " $O/phase.log | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -m gpu -q -x -p no:cacheprovider -k "not cfg4" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cheb_step|k_fx_sym" -s 6 -c 3 \
    -o $O/full_cfg4 -f python tools/prof_step.py --config cfg4_3d_N128 --solves 1 > $O/ncu_cfg4.log 2>&1; echo ncu cfg4=$?
