# ncu --set full of the matrix-free K12 (direct engine) and K3 (staged engine),
# config 2, exported to CSV (the .ncu-rep stays in /tmp: too large to copy back)
TAG=${1:-s1}
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil -s 5 -c 2 \
  -o /tmp/${TAG}_stencil -f python tools/prof_solve.py --operator stencil --iters 10 > $O/ncu_stencil_$TAG.log 2>&1
ncu -i /tmp/${TAG}_stencil.ncu-rep --page details --csv > $O/${TAG}_stencil_details.csv 2>&1
ncu -i /tmp/${TAG}_stencil.ncu-rep --page raw --csv > $O/${TAG}_stencil_raw.csv 2>&1
ncu -i /tmp/${TAG}_stencil.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_stencil_source.csv 2>/dev/null
python tools/ncu_hot_sass.py /tmp/${TAG}_stencil_source.csv > $O/${TAG}_stencil_hot_sass.txt 2>&1
ls -la /tmp/${TAG}_stencil.ncu-rep /tmp/${TAG}_stencil_source.csv
