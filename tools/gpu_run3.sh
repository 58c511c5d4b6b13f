mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gemm_lab3 tools/gemm_lab3.cu && ./tools/gemm_lab3 > gpurun_out/lab3b.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pdl.json 2>gpurun_out/bench_pdl.err; echo b1=$?
DD_NO_PDL=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nopdl.json 2>gpurun_out/bench_nopdl.err; echo b2=$?
