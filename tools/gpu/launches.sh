#!/bin/bash
# usage: tools/gpu/launches.sh <out.csv> <command...>   (one launch list: device time + DRAM bytes per kernel)
out=$1; shift
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file "$out" "$@" > /dev/null 2>&1
