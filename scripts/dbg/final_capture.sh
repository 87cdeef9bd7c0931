set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02g_pytest.log 2>&1; tail -2 gpurun_out/r02g_pytest.log
python bench.py --impl reference > gpurun_out/r02g_reference.json 2> gpurun_out/r02g_reference.err
python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
python bench.py --workload config4 > gpurun_out/r02g_bench_c4.json 2> gpurun_out/r02g_bench_c4.err
REPS=3 ncu --set full --clock-control none --import-source on -k regex:k_eval_staged -s 3 -c 1 -f -o gpurun_out/r02g_c3 python scripts/kbench.py > gpurun_out/r02g_ncu_c3.log 2>&1
WORKLOAD=config4 REPS=3 ncu --set full --clock-control none --import-source on -k regex:k_eval_staged -s 3 -c 1 -f -o gpurun_out/r02g_c4 python scripts/kbench.py > gpurun_out/r02g_ncu_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02g_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-single > gpurun_out/r02g_launches.log 2>&1
ls -la gpurun_out/r02g*
