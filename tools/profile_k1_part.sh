# ncu --set full of the multi-GPU schedule's K1 (plain As = A s, EpiStore) and K3 at N = 1
TAG=${1:-k1p}
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr_pipe_kernel -s 4 -c 2 \
  -o /tmp/${TAG} -f python bench.py --partitioned --no-cpu --steps 1 --warmup 3 > $O/ncu_$TAG.log 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page details --csv > $O/${TAG}_details.csv 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_source.csv 2>/dev/null
python tools/ncu_hot_sass.py /tmp/${TAG}_source.csv > $O/${TAG}_hot_sass.txt 2>&1
