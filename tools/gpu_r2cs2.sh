# class-sparse vs dense-block H̃ stream on cfg4 (tool; under gpurun from the repo root)
mkdir -p gpurun_out/cs2
O=gpurun_out/cs2
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
for v in 1 0; do
  DD_FX_CLASS_SPARSE=$v timeout 900 python bench.py --config cfg4_3d_N128 --no-cpu-baseline > $O/bench_cfg4_cs$v.json 2> $O/bench_cfg4_cs$v.err; echo b4 cs$v=$?
  DD_NO_GRAPH=1 DD_FX_CLASS_SPARSE=$v timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:"k_fx_sym" \
    -s 20 -c 12 --log-file $O/fx_cs$v.csv python tools/prof_step.py --config cfg4_3d_N128 --solves 2 > $O/ncu_fx_cs$v.log 2>&1; echo ncufx=$?
done
export DD_NO_GRAPH=1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cheb_step|k_fx_sym" -s 40 -c 3 \
    -o $O/full_cfg4 -f python tools/prof_step.py --config cfg4_3d_N128 --solves 2 > $O/ncu_cfg4.log 2>&1; echo ncu=$?
