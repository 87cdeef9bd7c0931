# dev probe: DRAM bytes of k_eval_staged under both processing orders
for o in bus tree; do
 for w in config3 config4; do
 PF_ORDER=$o WORKLOAD=$w REPS=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_eval_staged -s 3 -c 1 --csv --log-file gpurun_out/order_$o_$w.csv python scripts/kbench.py > /dev/null 2>&1
 echo "$o $w"; python - "gpurun_out/order_$o_$w.csv" <<'P'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r)); print(d.get('Metric Name'),d.get('Metric Unit'),d.get('Metric Value'))
P
 done
done
