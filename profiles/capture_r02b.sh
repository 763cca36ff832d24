#!/bin/bash
# Round-2 captures after the grouped K1 column lists (one B200 under gpurun;
# never a multi-rank command). Same recipe as capture_r02.sh.
set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
O=gpurun_out/prof
mkdir -p $O
# 1. K1 SpMV, config 2 (grouped 16-bit columns): 20 launches
ncu --metrics $M --clock-control none -k regex:"k1_(stream_)?kernel" -s 5 -c 20 --csv --log-file $O/r02b_ncu_k1_c2_launches.csv \
    python bench.py --steps 30 --warmup 3 --no-cpu-baseline --cg-steps 0 > /dev/null 2>&1
# 2. partitioned CG on the whole config 5 (grouped int32 columns): 10 live iterations' kernels
ncu --metrics $M --clock-control none -k regex:"k1_dot|dot_final|update_kernel|p_kernel|pq_kernel" -s 40 -c 40 --csv \
    --log-file $O/r02b_ncu_cg_c5_launches.csv \
    python bench.py --workload cg --config c5 --steps 1 --warmup 1 --iterations 50 --no-cpu-baseline > /dev/null 2>&1
# 3. full sections of the grouped K1 on config 2
ncu --set full --import-source on --clock-control none -k regex:"k1_(stream_)?kernel" -s 5 -c 1 -o $O/r02b_k1_c2_grouped_full \
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --cg-steps 0 > /dev/null 2>&1
ls -la $O
# 4. (later in round 2b) CG iteration kernels, config 4 locality order, after the update / p prefetch
ncu --metrics $M --clock-control none -k regex:"k1_dot|dot_final|update_kernel|p_kernel" -s 80 -c 40 --csv \
    --log-file $O/r02b_ncu_cg_c4_locality_launches.csv \
    python bench.py --workload cg --steps 1 --warmup 3 --iterations 50 --both-orders 0 --no-cpu-baseline > /dev/null 2>&1
# 5. K2 on accelerator in 128-thread CTAs at T = 20 (full sections)
ncu --set full --import-source on --clock-control none -k regex:k2_kernel -c 1 -o $O/r02b_k2_accel_full \
    python profiles/suite_once.py accelerator k2:20 > /dev/null 2>&1
# 6. config 3 suite: one launch of K1 / K1rs / K2 (T 16, 20, 32) per matrix with the round-2b kernels
ncu --metrics $M --clock-control none -k regex:"k1_|k2_kernel" --csv --log-file $O/r02b_ncu_suite_launches.csv \
    python profiles/suite_once.py "" k1,k1rs,k2:16,k2:20,k2:32 > /dev/null 2>&1
