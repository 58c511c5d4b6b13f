# Quick GPU check (tool; under gpurun from the repo root): build, selected -m gpu tests ($TESTS),
# then bench lines for $CONFIGS with extra env settings from $ENVS (";"-separated, "-" = none).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c_build.log 2>&1; echo build=$?
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest $TESTS -m gpu -x -q > gpurun_out/c_pytest.log 2>&1; echo pytest=$?; fi
IFS=';' read -ra EV <<< "${ENVS:--}"
for c in $CONFIGS; do for e in "${EV[@]}"; do
  tag=$(echo "$e" | tr -c 'A-Za-z0-9_\n' '_')
  if [ "$e" = "-" ]; then e=""; fi
  env $e timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline $BENCH_ARGS > gpurun_out/c_bench_${c}_${tag}.json 2>&1; echo bench $c $tag=$?
done; done
