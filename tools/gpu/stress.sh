for rep in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py tests/test_gpu_fuzz.py -q -p no:randomly 2>&1 | tail -1; done
for rep in 1 2 3; do for W in "1,1" "2,2" "1,2"; do PDG_LATTICE_WARPS=$W timeout 300 python -m pytest tests/test_gpu_lattice.py -q -k "transport and N33" 2>&1 | tail -1; done; done
