# tagged y-trace hand-over: lattice parity, then the lattice workloads + launch list
timeout 1200 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py -q -x > gpurun_out/lly_pytest.txt 2>&1
for L in D3Q15 D3Q19 D3Q27; do timeout 300 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lly_$L.json 2> gpurun_out/lly_$L.err; done
timeout 300 python bench.py --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lly_D2Q9.json 2> gpurun_out/lly_D2Q9.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lly_D3Q27.csv python bench.py --lattice D3Q27 --cells 128 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
