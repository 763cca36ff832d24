#!/bin/bash
# Round-2 ncu captures behind profiles/ (one B200 under gpurun; never a
# multi-rank command). Launch lists: --metrics pass, cold caches unless
# --cache-control none, serialised launches: compare SHARES with the bench's
# CUDA-event numbers, not absolutes.
set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
O=gpurun_out/prof
mkdir -p $O
# 1. K1 SpMV, config 2 (the default bench's headline kernel): 20 launches
ncu --metrics $M --clock-control none -k regex:"k1_(stream_)?kernel" -s 5 -c 20 --csv --log-file $O/r02_ncu_k1_c2_launches.csv \
    python bench.py --steps 30 --warmup 3 --no-cpu-baseline --cg-steps 0 > /dev/null 2>&1
# 2. CG iteration kernels, config 4, both row orders (skip into the first solve's live iterations)
for ORD in locality reference; do
ncu --metrics $M --clock-control none -k regex:"k1_dot|dot_final|update_kernel|p_kernel" -s 80 -c 40 --csv \
    --log-file $O/r02_ncu_cg_c4_${ORD}_launches.csv \
    python bench.py --workload cg --steps 1 --warmup 3 --iterations 50 --row-order $ORD --both-orders 0 --no-cpu-baseline > /dev/null 2>&1
done
# 3. partitioned CG on the whole config 5 (one partition = one GPU): 10 live iterations' kernels
ncu --metrics $M --clock-control none -k regex:"k1_dot|dot_final|update_kernel|p_kernel|pq_kernel" -s 40 -c 40 --csv \
    --log-file $O/r02_ncu_cg_c5_launches.csv \
    python bench.py --workload cg --config c5 --steps 1 --warmup 1 --iterations 50 --no-cpu-baseline > /dev/null 2>&1
# 4. config 3 suite: one launch of K1 / K1rs / K2 per matrix (the K1 for few long rows included)
ncu --metrics $M --clock-control none -k regex:"k1_|k2_kernel" --csv --log-file $O/r02_ncu_suite_launches.csv \
    python profiles/suite_once.py "" k1,k1rs,k2:8,k2:16 > /dev/null 2>&1
# 5. full sections: the few-long-rows K1 on protein, the CG SpMV+p.q on config 4 (locality)
ncu --set full --import-source on --clock-control none -k regex:k1_coop -c 1 -o $O/r02_k1coop_protein_full \
    python profiles/suite_once.py protein k1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k1_dot -s 20 -c 1 -o $O/r02_k1dot_c4_locality_full \
    python bench.py --workload cg --steps 1 --warmup 3 --iterations 50 --both-orders 0 --no-cpu-baseline > /dev/null 2>&1
ls -la $O
