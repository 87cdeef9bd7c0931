# dev probe: L2 cache hints as immediate descriptors (time and DRAM bytes)
AB_C4=1 scripts/ab_libs.sh "$@"
for lib in "$@"; do
 v=$(basename $lib .so)
 PFGPU_LIB=$lib REPS=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_eval_staged -s 3 -c 1 --csv --log-file gpurun_out/hint_$v.csv python scripts/kbench.py > /dev/null 2>&1
 echo "$v $(grep -E 'dram__bytes' gpurun_out/hint_$v.csv | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' ')"
done
