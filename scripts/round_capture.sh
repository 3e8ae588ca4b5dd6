set -x
python -m pytest tests -m gpu -q > gpurun_out/k_tests.log 2>&1; tail -2 gpurun_out/k_tests.log
timeout 1500 python tests/tools/fuzz_parity.py 400 29 > gpurun_out/k_fuzz.log 2>&1; tail -2 gpurun_out/k_fuzz.log
timeout 900 python tests/tools/parity_sweep.py 64 > gpurun_out/k_sweep.log 2>&1; tail -4 gpurun_out/k_sweep.log
python bench.py > gpurun_out/k_bench.json 2> gpurun_out/k_bench.err; head -c 400 gpurun_out/k_bench.json
python bench.py --impl reference > gpurun_out/k_ref.json 2> gpurun_out/k_ref.err; head -c 300 gpurun_out/k_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --inflight 1 > gpurun_out/k_ncu.log 2>&1; echo ncu $?
ncu --set full --import-source on --clock-control none --kernel-name-base function -k k_star --launch-skip 1 -c 1 -o gpurun_out/k_full python scripts/pipeline_once.py 64 > gpurun_out/k_full.log 2>&1; echo full $?
