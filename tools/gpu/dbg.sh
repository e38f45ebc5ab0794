for N in 16 33 64 128; do for L in D3Q19 D3Q27; do timeout 120 python tools/gpu/dbg_lat.py $L $N 0 2>&1 | tail -1; timeout 120 python tools/gpu/dbg_lat.py $L $N 3 2>&1 | tail -1; done; done
timeout 600 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py -q 2>&1 | tail -3
