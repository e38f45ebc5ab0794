set -x
timeout 600 python -m pytest tests/test_gpu_lattice.py -q -x 2>&1 | tail -2
for L in D3Q27 D3Q19 D3Q15; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e > gpurun_out/lat_bench_$L.json 2> gpurun_out/lat_bench_$L.err; done
timeout 600 python bench.py --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e > gpurun_out/lat_bench_D2Q9.json 2> gpurun_out/lat_bench_D2Q9.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lat_launches_D3Q27.csv python bench.py --lattice D3Q27 --cells 128 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
