#!/bin/bash
# Export an ncu report into small csv files next to it and delete the report (the
# gpurun merge-back limit is 64 MiB).  usage: scripts/ncu_export.sh gpurun_out/prof_X.ncu-rep
rep=$1; base=${rep%.ncu-rep}
ncu -i "$rep" --page details --csv > ${base}_details.csv 2>/dev/null
ncu -i "$rep" --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active > ${base}_raw.csv 2>/dev/null
ncu -i "$rep" --page source --csv -k regex:interp_tile > ${base}_src_interp.csv 2>/dev/null
grep -c UTMALDG ${base}_src_interp.csv > ${base}_utmaldg_count.txt
ncu -i "$rep" --page source --csv -k regex:spread_outer > ${base}_src_spread.csv 2>/dev/null
[ -s ${base}_src_spread.csv ] && python scripts/ncu_sass_summary.py ${base}_src_spread.csv 25 > ${base}_sass_spread.txt
[ -s ${base}_src_interp.csv ] && python scripts/ncu_sass_summary.py ${base}_src_interp.csv 25 > ${base}_sass_interp.txt
gzip -f ${base}_src_interp.csv ${base}_src_spread.csv
rm -f "$rep"
