# Full GPU check (tool; run under gpurun from the repo root): build, the -m gpu suite, smoke, then
# the evidence pass of gpu_profile_r1.sh.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r_build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r_pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1; echo smoke=$?
bash tools/gpu_profile_r1.sh
