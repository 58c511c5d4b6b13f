mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for pdl in 0 1; do
DD_NO_PDL=$pdl timeout 300 python bench.py --config cfg3_2d_N4096 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench5_nopdl$pdl.json 2>&1; echo b=$?
done
