# Round-2 evidence on the sliced-ELL build (one B200): bench lines of every
# workload, the reference arm, the ncu launch list of the default bench, ncu
# --set full captures of config 2's and config 4's K12 + K3 (with the
# per-instruction stall samples of config 2), the schedule evidence logs, and
# the plain-dot measurement build.  Usage: bash tools/profile_r2b.sh OUTDIR
O=${1:-gpurun_out/r2b}
mkdir -p $O $O/evidence
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { name=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo "bench $name rc=$?"; }
run c2 --steps 20 --warmup 5
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>/dev/null; echo "reference rc=$?"
run c2_stencil --operator stencil --steps 10 --warmup 3 --no-cpu
run c2_part --partitioned --steps 10 --warmup 3 --no-cpu
run c2_part_stencil --partitioned --operator stencil --steps 10 --warmup 3 --no-cpu
run c2_lb2 --loopback 2 --steps 5 --warmup 3
run c2_lb4 --loopback 4 --steps 5 --warmup 3
run c4 --config c4 --steps 3 --warmup 3 --no-cpu
run c4_stencil --config c4 --operator stencil --steps 5 --warmup 3 --no-cpu
run c4_part --config c4 --partitioned --steps 3 --warmup 3
run c4_part_stencil --config c4 --operator stencil --partitioned --steps 5 --warmup 3
run c4_lb8 --config c4 --loopback 8 --steps 2 --warmup 3
if [ -f paper_2108_10591_b200/variants/libpbsafe_plaindot.so ]; then
  PBS_LIB=$PWD/paper_2108_10591_b200/variants/libpbsafe_plaindot.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-comparators > $O/bench_c2_plaindot.json 2>/dev/null; echo "plaindot rc=$?"
fi
timeout 1500 python tools/run_configs.py --out $O/configs.json > $O/configs.log 2>&1; echo "configs rc=$?"
timeout 600 python tools/schedule_evidence.py $O/evidence > $O/evidence.log 2>&1; echo "evidence rc=$?"
# launch list of the default bench workload (cold-cache, serialised: shares)
python bench.py --steps 1 --warmup 1 --no-cpu --no-comparators > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/c2_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-comparators > $O/ncu_launches.log 2>&1
echo "launches rc=$?"
bash tools/profile_sell.sh $O c2
python tools/ncu_regions.py $O/c2_k12_k3_source.csv.gz > $O/c2_wait_sites.txt 2>&1
python tools/prof_solve.py --config c4 --operator devcsr --iters 3 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sell_pipe_kernel -s 4 -c 2 \
  -o /tmp/c4_k12_k3 -f python tools/prof_solve.py --config c4 --operator devcsr --iters 3 > $O/ncu_c4.log 2>&1
ncu -i /tmp/c4_k12_k3.ncu-rep --page details --csv > $O/c4_k12_k3_details.csv 2>&1
ncu -i /tmp/c4_k12_k3.ncu-rep --page raw --csv > $O/c4_k12_k3_raw.csv 2>&1
echo done
