timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lat_launches_D3Q27_v2.csv python bench.py --lattice D3Q27 --cells 128 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lat_launches_D2Q9_v2.csv python bench.py --lattice D2Q9 --cells 1024 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
