timeout 600 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py -q -x 2>&1 | tail -2
for L in D3Q27 D3Q19; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/rl_a_$L.json 2>&1; done
cp paper_1702_00169_b200/libpdg_lb2.so paper_1702_00169_b200/libpdg.so
for L in D3Q27 D3Q19; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/rl_b_$L.json 2>&1; done
echo done
