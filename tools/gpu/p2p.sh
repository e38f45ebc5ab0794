timeout 900 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -2
for W in "1,1" "2,2" "1,2"; do PDG_LATTICE_WARPS=$W timeout 300 python -m pytest tests/test_gpu_lattice.py -q -x -k "transport" 2>&1 | tail -1; done
for L in D3Q15 D3Q19 D3Q27; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p2p_$L.json 2>&1; done
echo done
