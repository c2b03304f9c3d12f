#!/bin/bash
# usage: scripts/ncu_details.sh REP [kernel-regex]
ncu -i "$1" --page details --csv ${2:+-k regex:$2} 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
want=['Duration','DRAM Throughput','Memory Throughput','Compute (SM) Throughput','Achieved Occupancy','Theoretical Occupancy','Registers Per Thread','Dynamic Shared Memory Per Block','Block Limit Shared Mem','Block Limit Registers','L1/TEX Hit Rate','L2 Hit Rate','Executed Ipc Active','Issue Slots Busy','Achieved Active Warps Per SM','Elapsed Cycles','SM Frequency']
for row in r[1:]:
    if row[mi] in want: print(row[ki][:38], '|', row[mi], row[vi], row[ui])
"
