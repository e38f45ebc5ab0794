# per-launch ncu lists of the lattice workloads (current build)
for L in D3Q15 D3Q19 D3Q27; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lat4_$L.csv python bench.py --lattice $L --cells 128 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lat4_D2Q9.csv python bench.py --lattice D2Q9 --cells 1024 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
