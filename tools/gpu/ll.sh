# tagged x-trace hand-over: lattice parity, then the lattice workloads
timeout 1200 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py -q -x > gpurun_out/ll_pytest.txt 2>&1
for N in 1024 2048; do timeout 300 python bench.py --lattice D2Q9 --cells $N --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ll_D2Q9_$N.json 2> gpurun_out/ll_D2Q9_$N.err; done
for L in D3Q15 D3Q19 D3Q27; do timeout 300 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ll_$L.json 2> gpurun_out/ll_$L.err; done
echo done
