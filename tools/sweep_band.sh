# band mode (config 3) with more staged products in flight per row at 1 CTA/SM
runt() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 20 --timing --repeat 2 $2 2>&1 | tail -1)"; }
runt "" "--config c3"
runt "PBS_LIB=paper_2108_10591_b200/variants/libpbsafe_band4.so" "--config c3"
runt "PBS_LIB=paper_2108_10591_b200/variants/libpbsafe_band8.so" "--config c3"
