# x written back by the freezing kernel (pinned host x): tests + e2e A/B against the copy after the loop.
mkdir -p gpurun_out/g5; O=gpurun_out/g5
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "pinned or host" > $O/pytest.log 2>&1; echo pytest=$?
tail -3 $O/pytest.log
for c in cfg5_2d_N2048_darcy cfg2_2d_N1024_sweep; do
  for z in 0 1 0 1; do
    [ $z = 1 ] && export DD_NO_ZERO_COPY=1 || unset DD_NO_ZERO_COPY
    timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_z$z.json 2> $O/bench_${c}_z$z.err
    python -c "import json;d=json.load(open('$O/bench_${c}_z$z.json'));print('$c nozc=$z', d['value'], d['e2e'])"
  done
done
unset DD_NO_ZERO_COPY
