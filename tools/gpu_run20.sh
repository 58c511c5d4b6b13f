mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export DD_NO_GRAPH=1
timeout 600 python bench.py --config cfg4_3d_N128 --steps 1 --warmup 3 > gpurun_out/p20_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dgemm|k_inner|k3_|k_face|k_gather|k_pcg3" -s 100 -c 400 --csv \
  --log-file gpurun_out/p20_launches_cfg4.csv python bench.py --config cfg4_3d_N128 --steps 1 --warmup 3 > gpurun_out/p20_ncu.log 2>&1; echo ncu=$?
