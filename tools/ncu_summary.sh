#!/bin/bash
# usage: tools/ncu_summary.sh report.ncu-rep  -> key metrics of every profiled kernel
ncu -i "$1" --page details --csv 2>/dev/null | python3 -c '
import csv, sys
keep = {"Duration","DRAM Throughput","Memory Throughput","Compute (SM) Throughput","SM Frequency","Executed Ipc Active",
 "Issue Slots Busy","Registers Per Thread","Achieved Occupancy","Theoretical Occupancy","Executed Instructions",
 "Active Warps Per Scheduler","Eligible Warps Per Scheduler","No Eligible","L1/TEX Hit Rate","L2 Hit Rate","Max Bandwidth","Mem Pipes Busy","Grid Size","Block Size","Warp Cycles Per Issued Instruction"}
for row in csv.reader(sys.stdin):
    if len(row) < 12 or row[0] == "ID": continue
    name = row[-4] if False else None
    metric, unit, val = row[12], row[13], row[14]
    if metric in keep: print(f"{row[4][:40]:40s} {metric:38s} {val:>16s} {unit}")
'
