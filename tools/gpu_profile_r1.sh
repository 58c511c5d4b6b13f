# Round-1 evidence pass (tool; run under gpurun from the repo root): bench lines for every
# workload, the ncu launch list of the headline bench command, one full ncu capture of the
# dominant kernels.  Outputs land in gpurun_out/ and are summarised into profiles/ by hand.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/p_gpu.txt
for c in cfg2_2d_N1024_sweep cfg3_2d_N4096 cfg5_2d_N2048_darcy cfg1_2d_N32 cfg4_3d_N128 cfg5i_2d_N2048_darcy_rtol1e-5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/p_bench_$c.json 2> gpurun_out/p_bench_$c.err; echo bench $c=$?
done
timeout 600 python bench.py --frac-mode ra --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/p_bench_cfg2_ra.json 2>&1; echo ra=$?
timeout 900 python bench.py --mode bulk --steps 3 --warmup 1 > gpurun_out/p_bench_cfg2_bulk.json 2>&1; echo bulk=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/p_bench_ref_cfg2.json 2>&1; echo ref=$?
# ncu launch list of the headline command (cold-cache, serialised: shares, not absolutes)
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/p_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p_ncu_launch.log 2>&1; echo ncu1=$?
# NEXT rows: RA-evaluated F in 3D, bulk PCG with the Eq.(5) preconditioner, general t
timeout 900 python bench.py --config cfg4_3d_N128 --frac-mode ra --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p_bench_cfg4_ra.json 2>&1; echo cfg4ra=$?
timeout 900 python bench.py --mode bulk-pcg --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p_bench_cfg2_bulkpcg.json 2>&1; echo bpcg=$?
timeout 600 python bench.py --t 0.25 --shifted --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/p_bench_cfg2_t025.json 2>&1; echo t025=$?
# NEXT-1 in 3D: bulk solves, the bulk PCG, and Remark 1's RA-operator bulk PCG
timeout 900 python bench.py --config cfg4_3d_N128 --mode bulk --steps 3 --warmup 2 > gpurun_out/p_bench_cfg4_bulk.json 2>&1; echo cfg4bulk=$?
timeout 900 python bench.py --config cfg4_3d_N128 --mode bulk-pcg --steps 2 --warmup 1 > gpurun_out/p_bench_cfg4_bulkpcg.json 2>&1; echo cfg4bpcg=$?
timeout 900 python bench.py --config cfg4_3d_N128 --mode bulk-pcg --frac-mode ra --steps 2 --warmup 1 > gpurun_out/p_bench_cfg4_bulkpcg_ra.json 2>&1; echo cfg4bpcgra=$?
