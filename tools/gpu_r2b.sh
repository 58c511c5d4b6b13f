# round-2 bulk / bulk-PCG bench lines (NEXT-1) and the factored / assembled 2D Schur modes
mkdir -p gpurun_out/ev2
O=gpurun_out/ev2
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
for c in cfg2_2d_N1024_sweep cfg4_3d_N128; do
  for m in bulk bulk-pcg; do
    timeout 1500 python bench.py --config $c --mode $m --no-cpu-baseline > $O/bench_${c}_$m.json 2> $O/bench_${c}_$m.err; echo $c $m=$?
  done
done
timeout 1500 python bench.py --config cfg4_3d_N128 --mode bulk-pcg --frac-mode ra --no-cpu-baseline > $O/bench_cfg4_bulk-pcg_ra.json 2> $O/bench_cfg4_bulk-pcg_ra.err; echo cfg4 bulkpcg ra=$?
for s in factored assembled; do
  timeout 900 python bench.py --schur $s --no-cpu-baseline > $O/bench_cfg5_$s.json 2> $O/bench_cfg5_$s.err; echo cfg5 $s=$?
done
