# Round-2 evidence run on one B200: bench lines of every workload, the ncu
# launch list of the default bench, and ncu --set full captures (exported as
# CSV) of the hot kernels: config-2 K12 + K3 (CSR, fused single-GPU
# schedule), config-4 matrix-free K12 + K3 (z-marching engine), and the plain
# CSR SpMV (the multi-GPU schedule's K1).  Usage: bash tools/profile_r2.sh OUTDIR
O=${1:-gpurun_out/r2}
mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { name=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo "bench $name rc=$?"; }
run c2 --steps 20 --warmup 5
run c2_stencil --operator stencil --steps 10 --warmup 3 --no-cpu
run c2_part --partitioned --steps 10 --warmup 3
run c2_part_stencil --partitioned --operator stencil --steps 10 --warmup 3
run c2_lb2 --loopback 2 --steps 5 --warmup 3
run c2_lb4 --loopback 4 --steps 5 --warmup 3
run c4 --config c4 --steps 3 --warmup 3 --no-cpu
run c4_stencil --config c4 --operator stencil --steps 5 --warmup 3 --no-cpu
run c4_part --config c4 --partitioned --steps 3 --warmup 3
run c4_part_stencil --config c4 --operator stencil --partitioned --steps 5 --warmup 3
run c4_lb8 --config c4 --loopback 8 --steps 2 --warmup 3
run c4_lb8_stencil --config c4 --operator stencil --loopback 8 --steps 3 --warmup 3
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>/dev/null; echo "reference rc=$?"
# launch list of the default bench workload (cold-cache, serialised: shares)
python bench.py --steps 1 --warmup 1 --no-cpu --no-comparators > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/c2_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-comparators > $O/ncu_launches.log 2>&1
echo "launches rc=$?"
# full captures
python tools/prof_solve.py --iters 10 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr_pipe_kernel -s 6 -c 2 \
  -o /tmp/c2_k12_k3 -f python tools/prof_solve.py --iters 10 > $O/ncu_c2.log 2>&1
ncu -i /tmp/c2_k12_k3.ncu-rep --page details --csv > $O/c2_k12_k3_details.csv 2>&1
ncu -i /tmp/c2_k12_k3.ncu-rep --page raw --csv > $O/c2_k12_k3_raw.csv 2>&1
python tools/prof_solve.py --config c4 --operator stencil --iters 3 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_zm_kernel -s 4 -c 2 \
  -o /tmp/c4s_k12_k3 -f python tools/prof_solve.py --config c4 --operator stencil --iters 3 > $O/ncu_c4s.log 2>&1
ncu -i /tmp/c4s_k12_k3.ncu-rep --page details --csv > $O/c4s_k12_k3_details.csv 2>&1
ncu -i /tmp/c4s_k12_k3.ncu-rep --page raw --csv > $O/c4s_k12_k3_raw.csv 2>&1
PBS_PLAIN_TPR=0 python tools/csr_micro.py c2 3 > /dev/null 2>&1 && PBS_PLAIN_TPR=0 \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_pipe_kernel -s 2 -c 1 \
  -o /tmp/c2_k1 -f python tools/csr_micro.py c2 3 > $O/ncu_k1.log 2>&1
ncu -i /tmp/c2_k1.ncu-rep --page details --csv > $O/c2_k1_plain_details.csv 2>&1
ncu -i /tmp/c2_k1.ncu-rep --page raw --csv > $O/c2_k1_plain_raw.csv 2>&1
echo done
