# ncu --set full of config 3's K12 and K3 (band-mode CSR engine), CSV exports
TAG=${1:-c3a}
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr_pipe_kernel -s 2 -c 2 \
  -o /tmp/${TAG} -f python tools/prof_solve.py --config c3 --iters 3 > $O/ncu_$TAG.log 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page details --csv > $O/${TAG}_details.csv 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_source.csv 2>/dev/null
python tools/ncu_hot_sass.py /tmp/${TAG}_source.csv > $O/${TAG}_hot_sass.txt 2>&1
