# dev tool: the end-of-round capture (one gpurun call).  Stage 1: GPU tests and
# the ncu reports that profiles/traffic.json is made from (scripts/ncu_traffic.py,
# run in the build container); stage 2 (after traffic.json is updated): both
# bench arms, the config-4 bench line and the launch list.
set -x
if [ "$1" = ncu ]; then
python -m pytest tests -m gpu -x -q > gpurun_out/r02j_pytest.log 2>&1; tail -2 gpurun_out/r02j_pytest.log
REPS=3 ncu --set full --clock-control none --import-source on -k regex:k_eval_staged -s 3 -c 1 -f -o gpurun_out/r02j_c3 python scripts/kbench.py > gpurun_out/r02j_ncu_c3.log 2>&1
WORKLOAD=config4 REPS=3 ncu --set full --clock-control none --import-source on -k regex:k_eval_staged -s 3 -c 1 -f -o gpurun_out/r02j_c4 python scripts/kbench.py > gpurun_out/r02j_ncu_c4.log 2>&1
else
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j_smoke.log 2>&1; tail -1 gpurun_out/r02j_smoke.log
python bench.py --impl reference > gpurun_out/r02j_reference.json 2> gpurun_out/r02j_reference.err
python bench.py > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err
python bench.py --workload config4 --no-single > gpurun_out/r02j_bench_c4.json 2> gpurun_out/r02j_bench_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02j_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-single > gpurun_out/r02j_launches.log 2>&1
fi
ls -la gpurun_out/r02j*
