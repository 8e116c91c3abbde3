# Round profile of the bench workload (config 2 CSR): bench line, ncu launch
# list of the same command, one ncu --set full capture of K12 + K3 exported to
# CSV.  Usage: bash tools/profile_round.sh TAG
TAG=${1:-v7}
O=gpurun_out
timeout 600 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > $O/ncu_launches_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr_pipe_kernel -s 6 -c 2 \
  -o /tmp/${TAG}_k12_k3 -f python tools/prof_solve.py --iters 10 > $O/ncu_full_$TAG.log 2>&1
ncu -i /tmp/${TAG}_k12_k3.ncu-rep --page details --csv > $O/${TAG}_k12_k3_details.csv 2>&1
ncu -i /tmp/${TAG}_k12_k3.ncu-rep --page raw --csv > $O/${TAG}_k12_k3_raw.csv 2>&1
ncu -i /tmp/${TAG}_k12_k3.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_k12_k3_source.csv 2>/dev/null
python tools/ncu_hot_sass.py /tmp/${TAG}_k12_k3_source.csv > $O/${TAG}_k12_k3_hot_sass.txt 2>&1
ls -la /tmp/${TAG}_k12_k3.ncu-rep
# the report itself stays on the box: gpurun copies back at most 64 MiB
