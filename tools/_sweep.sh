python -m pytest tests/test_gpu_gap.py -x -q 2>&1 | tail -2
timeout 400 python tools/stress_gap.py 3000 111 2>&1 | tail -3
run() { timeout 300 python tools/gap_check.py $1 $2 $3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config'], d['n_sets'], d['n_hash'], round(d['ms_visit'],4), round(d['ms_gap'],4), d['equal'], d['oracle_rows_equal'])"; }
run cfg4 2000000; run cfg4 2000000; run cfg3 400000; run cfg4 100000 4096
