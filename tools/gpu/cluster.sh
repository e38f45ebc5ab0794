timeout 600 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py -q -x 2>&1 | tail -4
for CS in 1 2 4 8; do for L in D3Q15 D3Q19 D3Q27; do PDG_LATTICE_CLUSTER=$CS timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/cl${CS}_$L.json 2>&1; done; done
PDG_LATTICE_CLUSTER=8 timeout 600 python -m pytest tests/test_gpu_lattice.py -q -x -k "transport and w1" 2>&1 | tail -2
echo done
