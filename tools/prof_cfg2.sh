# GPU profiling pass for the config-2 path (tool; run under gpurun from the repo root)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gemm_lab tools/gemm_lab.cu -lcublas
timeout 300 ./tools/gemm_lab 3 > gpurun_out/lab_cfg2.jsonl 2>&1; echo lab=$?
DD_PHASE_TIMING=1 timeout 120 python tools/prof_step.py --solves 3 > gpurun_out/phase_cfg2.log 2>&1; echo phase=$?
export DD_NO_GRAPH=1
timeout 120 python tools/prof_step.py --solves 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dgemm_tile|k_pcg_iter" -s 6 -c 3 \
    -o gpurun_out/prof_cfg2 -f python tools/prof_step.py --solves 2 > gpurun_out/ncu_cfg2.log 2>&1; echo ncu=$?
