mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export DD_NO_GRAPH=1
timeout 120 python tools/prof_step.py --solves 2 > gpurun_out/p_plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_dgemm_tile|k_pcg_iter" -s 6 -c 3 \
    -o gpurun_out/p_full_cfg2 -f python tools/prof_step.py --solves 2 > gpurun_out/p_ncu_full.log 2>&1; echo ncu=$?
