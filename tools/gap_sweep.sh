python -m pytest tests/test_gpu_gap.py -x -q 2>&1 | tail -2
for s in 31 32; do timeout 400 python tools/stress_gap.py 6000 $s 2>&1 | tail -3; done
