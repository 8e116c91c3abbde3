# ncu --set full capture of the sliced-ELL K12 + K3 (config 2 CSR) with the
# per-instruction stall samples.  Usage: bash tools/profile_sell.sh OUTDIR TAG
O=${1:-gpurun_out/sell}; TAG=${2:-sell}
mkdir -p $O
python tools/prof_solve.py --iters 10 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sell_pipe_kernel -s 6 -c 2 \
  -o /tmp/${TAG}_k12_k3 -f python tools/prof_solve.py --iters 10 > $O/ncu_full_$TAG.log 2>&1
ncu -i /tmp/${TAG}_k12_k3.ncu-rep --page details --csv > $O/${TAG}_k12_k3_details.csv 2>&1
ncu -i /tmp/${TAG}_k12_k3.ncu-rep --page raw --csv > $O/${TAG}_k12_k3_raw.csv 2>&1
ncu -i /tmp/${TAG}_k12_k3.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_k12_k3_source.csv 2>/dev/null
python tools/ncu_hot_sass.py /tmp/${TAG}_k12_k3_source.csv 60 > $O/${TAG}_k12_k3_hot_sass.txt 2>&1
gzip -c /tmp/${TAG}_k12_k3_source.csv > $O/${TAG}_k12_k3_source.csv.gz
