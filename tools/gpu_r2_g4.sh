# Compact pole-sum layout with the full smem carveout: resident CTAs per SM and the cfg5 A/B.
mkdir -p gpurun_out/g4; O=gpurun_out/g4
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
for w in 1 0 1 0; do
  [ $w = 0 ] && export DD_POLE_COMPACT=0 || unset DD_POLE_COMPACT
  DD_OCC_PRINT=1 timeout 300 python tools/time_precond.py --config cfg5_2d_N2048_darcy --reps 50 2>&1 | sort | uniq -c
  timeout 600 python bench.py --no-cpu-baseline > $O/bench_c$w.json 2> $O/bench_c$w.err; echo compact=$w rc=$?
  python -c "import json;d=json.load(open('$O/bench_c$w.json'));print('compact=$w', d['value'], d['e2e']['value'], d['roofline']['step']['frac'], d['roofline']['classes']['polesum_pcg']['measured_us'], d['roofline']['classes']['gemm_schur']['measured_us'])"
done
