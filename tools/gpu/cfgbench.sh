timeout 600 python -m pytest tests/test_gpu_lattice.py -q -x -k "N1 or N2" 2>&1 | tail -2
for C in 2 3 4; do timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/cfg$C.json 2> gpurun_out/cfg$C.err; done
echo done
