for L in D3Q15 D3Q19 D3Q27; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 > gpurun_out/final_$L.json 2> gpurun_out/final_$L.err; done
timeout 600 python bench.py --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 > gpurun_out/final_D2Q9.json 2> gpurun_out/final_D2Q9.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lat_launches_D3Q27_v3.csv python bench.py --lattice D3Q27 --cells 128 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
