#!/bin/bash
# ncu captures behind profiles/ (run on one B200 under gpurun; never a
# multi-rank command). Launch lists: --metrics pass, cold-cache and
# serialised, so compare SHARES with the bench's CUDA-event numbers.
set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
O=gpurun_out/prof
mkdir -p $O
# 1. K1 SpMV, config 2 (default bench): 20 launches, then one --set full
ncu --metrics $M --clock-control none -k regex:"k1_(stream_)?kernel" -s 5 -c 20 --csv --log-file $O/k1_c2_launches.csv \
    python bench.py --steps 30 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k1_(stream_)?kernel" -s 5 -c 1 -o $O/k1_c2_full \
    python bench.py --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# 2. K1 SpMV, config 1 (L2-resident)
ncu --metrics $M --clock-control none -k regex:k1_kernel -s 5 -c 10 --csv --log-file $O/k1_c1_launches.csv \
    python bench.py --config c1 --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# 3. CG iteration, config 4, locality order (k1rs): the CG kernels of 10 iterations, then k1_dot in full
# (one solve = one CUDA graph of 50 iterations; skip into the middle of the
# first solve so every captured launch is a live iteration)
ncu --metrics $M --clock-control none -k regex:"k1_dot|dot_final|update_kernel|p_kernel" -s 80 -c 40 --csv \
    --log-file $O/cg_c4_locality_launches.csv \
    python bench.py --workload cg --steps 1 --warmup 3 --iterations 50 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k1_dot -s 20 -c 1 -o $O/k1dot_c4_locality_full \
    python bench.py --workload cg --steps 1 --warmup 3 --iterations 50 --no-cpu-baseline > /dev/null 2>&1
# 4. same, reference row order
ncu --metrics $M --clock-control none -k regex:"k1_dot|dot_final|update_kernel|p_kernel" -s 80 -c 40 --csv \
    --log-file $O/cg_c4_reference_launches.csv \
    python bench.py --workload cg --steps 1 --warmup 3 --iterations 50 --row-order reference --no-cpu-baseline > /dev/null 2>&1
# 5. the CG kernels with warm caches (--cache-control none): the in-solve times
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none \
    -k regex:"k1_dot|dot_final|update_kernel|p_kernel" -s 80 -c 40 --csv --log-file $O/cg_c4_locality_warm_launches.csv \
    python bench.py --workload cg --steps 1 --warmup 3 --iterations 50 --no-cpu-baseline > /dev/null 2>&1
# 6. config 3 suite kernels (one launch each, every kernel id, each matrix)
ncu --metrics $M --clock-control none --csv --log-file $O/suite_launches.csv \
    python profiles/suite_once.py > /dev/null 2>&1
ls -la $O
