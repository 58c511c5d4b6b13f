mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for u in 1 2 4; do
DD_UNROLL=$u timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench17_u$u.json 2>&1; echo b=$?
done
