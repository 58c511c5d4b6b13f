# A/B: compact merged-interior pole-sum layout (3 CTAs/SM at cfg5) vs DD_POLE_COMPACT=0; parity.
mkdir -p gpurun_out/g3; O=gpurun_out/g3
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
for w in 1 0; do
  for c in cfg5_2d_N2048_darcy cfg5i_2d_N2048_darcy_rtol1e-5; do
    [ $w = 0 ] && export DD_POLE_COMPACT=0 || unset DD_POLE_COMPACT
    timeout 300 python tools/time_precond.py --config $c --reps 50 >> $O/precond.txt 2>&1
    timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_c$w.json 2> $O/bench_${c}_c$w.err; echo $c compact=$w rc=$?
    python -c "import json;d=json.load(open('$O/bench_${c}_c$w.json'));print('$c compact=$w', d['value'], d['e2e']['value'], d['roofline']['step'], d['roofline']['classes']['polesum_pcg'])"
  done
done
unset DD_POLE_COMPACT
cat $O/precond.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py tests/test_gpu_frac_ra.py tests/test_gpu_bulk.py -m gpu -q -x -p no:cacheprovider -k "not cfg4" > $O/pytest.log 2>&1; echo pytest=$?
tail -3 $O/pytest.log
for tool in memcheck synccheck racecheck; do
done
