cp paper_1702_00169_b200/libpdg.so /tmp/libpdg_new.so
for rep in 1 2; do
cp paper_1702_00169_b200/libpdg_head.so paper_1702_00169_b200/libpdg.so
timeout 600 python bench.py --lattice D3Q27 --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_head_$rep.json 2>&1
cp /tmp/libpdg_new.so paper_1702_00169_b200/libpdg.so
timeout 600 python bench.py --lattice D3Q27 --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_new_$rep.json 2>&1
done
echo done
