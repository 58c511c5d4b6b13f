mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke14.log 2>&1; echo smoke=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/torchrun14.json 2> gpurun_out/torchrun14.err; echo tr=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/torchrun14_ref.json 2> gpurun_out/torchrun14_ref.err; echo trref=$?
