# swizzled tensor-path buffers: lattice parity, then the 3-D lattice workloads
timeout 1200 python -m pytest tests/test_gpu_lattice.py -q -x > gpurun_out/swz_pytest.txt 2>&1
for L in D3Q15 D3Q27; do timeout 300 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/swz_$L.json 2> gpurun_out/swz_$L.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/swz_D3Q15.csv python bench.py --lattice D3Q15 --cells 128 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
