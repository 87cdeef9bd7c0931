# dev probe: time and DRAM bytes of k_eval_staged under both processing orders
for rep in 1 2 3; do for o in bus tree; do
  PF_ORDER=$o TAG="c3 order=$o" python scripts/kbench.py | tail -1
done; done
for rep in 1 2; do for o in bus tree; do
  PF_ORDER=$o WORKLOAD=config4 TAG="c4 order=$o" python scripts/kbench.py | tail -1
done; done
for o in bus tree; do for w in config3 config4; do
 PF_ORDER=$o WORKLOAD=$w REPS=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_eval_staged -s 3 -c 1 --csv --log-file gpurun_out/order_${o}_$w.csv python scripts/kbench.py > /dev/null 2>&1
 echo "$w order=$o $(grep -E 'dram__bytes' gpurun_out/order_${o}_$w.csv | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' ')"
done; done
