# ncu --set full of the multi-GPU schedule's kernels at N = 1 (K1 = As with the opportunistic block 1, K3) on
# config 2 and config 4 CSR.  Usage: bash tools/profile_part.sh OUTDIR
O=${1:-gpurun_out/part}; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for cfg in c2 c4; do
  python bench.py --config $cfg --partitioned --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:sell_pipe_kernel -s 40 -c 4 -o /tmp/part_$cfg -f \
    python bench.py --config $cfg --partitioned --steps 1 --warmup 1 --no-cpu > $O/ncu_part_$cfg.log 2>&1
  ncu -i /tmp/part_$cfg.ncu-rep --page details --csv > $O/part_${cfg}_details.csv 2>&1
  ncu -i /tmp/part_$cfg.ncu-rep --page raw --csv > $O/part_${cfg}_raw.csv 2>&1
  python tools/ncu_summary.py $O/part_${cfg}_details.csv | grep -E "sell_pipe|Duration|DRAM Thr|Memory Thr|Issue Slots|Grid Size"
done
