# Round-2 measurement set (run from the repo root on the GPU box); outputs under gpurun_out/r02.
set -x
mkdir -p gpurun_out/r02
python bench.py > gpurun_out/r02/bench_cfg4_default.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches_cfg4.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k _ZN3mhb11sign_kernelILi64ELb1ELb1EjLb0ELb0ELb1EEEvNS_8SignArgsEjjjj -c 1 -o gpurun_out/r02/sign_kernel_cfg4 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for c in cfg2 cfg3 cfg4; do python tools/scaling_projection.py $c 10 > gpurun_out/r02/scaling_projection_$c.json 2>/dev/null; done
python tools/scaling_projection.py cfg5 3 > gpurun_out/r02/scaling_projection_cfg5.json 2>/dev/null
python bench.py --config cfg2 --steps 20 --warmup 5 > gpurun_out/r02/bench_cfg2_iter.json 2>/dev/null
python bench.py --config cfg3 --steps 20 --warmup 5 --aux --no-e2e > gpurun_out/r02/bench_cfg3_iter_aux.json 2>/dev/null
python bench.py --config cfg3 --family random --steps 10 --warmup 3 --no-e2e > gpurun_out/r02/bench_cfg3_random.json 2>/dev/null
python bench.py --config cfg2 --family random --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/bench_cfg2_random.json 2>/dev/null
python bench.py --config cfg1 --steps 50 --warmup 5 > gpurun_out/r02/bench_cfg1_iter.json 2>/dev/null
python bench.py --config cfg1 --steps 50 --warmup 5 --graph --no-e2e --no-cpu-baseline > gpurun_out/r02/bench_cfg1_graph.json 2>/dev/null
python bench.py --config cfg1 --family random --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r02/bench_cfg1_random.json 2>/dev/null
ncu --metrics gpu__time_duration.sum,sm__cycles_active.max --clock-control none --csv --log-file gpurun_out/r02/launches_cfg1.csv python bench.py --config cfg1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python bench.py --config cfg4 --aux --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/bench_cfg4_aux.json 2>/dev/null
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02/bench_reference_arm.json 2>/dev/null
python bench.py --config c6 --steps 5 --warmup 2 > gpurun_out/r02/bench_c6.json 2>/dev/null
python bench.py --config cfg5 --steps 5 --warmup 3 > gpurun_out/r02/bench_cfg5_full_n1.json 2>/dev/null
python -m pytest tests -m gpu -q > gpurun_out/r02/pytest_gpu.log 2>&1
ls -la gpurun_out/r02
