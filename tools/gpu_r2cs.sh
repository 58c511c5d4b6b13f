# class-sparse H̃ stream check (tool; under gpurun from the repo root): r2/3D GPU tests, cfg4 bench,
# one ncu --set full capture of the packed stream + the fused Chebyshev step on cfg4
mkdir -p gpurun_out/cs
O=gpurun_out/cs
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_r2.py tests/test_gpu_3d.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest=$?
tail -2 $O/pytest.log
timeout 900 python bench.py --config cfg4_3d_N128 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo b4=$?
export DD_NO_GRAPH=1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cheb_step|k_fx_sym" -s 100 -c 3 \
    -o $O/full_cfg4 -f python tools/prof_step.py --config cfg4_3d_N128 --solves 1 > $O/ncu_cfg4.log 2>&1; echo ncu=$?
