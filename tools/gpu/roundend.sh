python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/re_ref.json 2> gpurun_out/re_ref.err; echo "ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/re_torchrun1.json 2> gpurun_out/re_torchrun1.err; echo "torchrun1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 5 --warmup 3 --decomp zslab --slabs-per-rank 4 --no-e2e --no-cpu-baseline > gpurun_out/re_torchrun1z.json 2> gpurun_out/re_torchrun1z.err; echo "torchrun1z rc=$?"
