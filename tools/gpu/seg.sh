# chain segments: parity tests, then the D2Q9 workloads
timeout 900 python -m pytest tests/test_gpu_lattice.py -q -x -k "segments or D2Q9 or fullsize" > gpurun_out/seg_pytest.txt 2>&1
for N in 1024 2048; do timeout 300 python bench.py --lattice D2Q9 --cells $N --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/seg_D2Q9_$N.json 2> gpurun_out/seg_D2Q9_$N.err; done
timeout 300 python bench.py --lattice-segment -1 --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/seg0_D2Q9_1024.json 2>&1
echo done
