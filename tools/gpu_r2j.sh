# grouped stream-K ring depth (tool)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/j_build.log 2>&1; echo build=$?
for v in 3 4 5; do for c in cfg5_2d_N2048_darcy cfg3_2d_N4096; do
  DD_GROUPED_PAIR=0 DD_GROUPED_STAGES=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/j_bench_s${v}_$c.json 2> gpurun_out/j_bench_s${v}_$c.err; echo bench $v $c=$?
done; done
