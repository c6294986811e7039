#!/bin/bash
# Steady-state DRAM traffic of K1: launches 31..42 of a 50-step run, no cache flush between them.
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum
CFGS=${CFGS:-"4_256 8_256 12_256 16_256 8_512 8_512_damp"}
for c in $CFGS; do
  cfg=$(echo $c | tr "_" " ")
  tag=$(echo $cfg | tr ' ' '_')
  timeout 600 ncu --cache-control none --clock-control none -k regex:k_tma -s 30 -c 12 --metrics $M --csv \
      python scripts/ncu_steady.py $cfg > gpurun_out/ncu_steady_$tag.csv 2> gpurun_out/ncu_steady_$tag.err
  echo "$cfg rc=$?"
done
