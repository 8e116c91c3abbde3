# staged products in flight per row in the 1-CTA instantiation: 8 (default) / 12 / 16
run() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 100 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
runt() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 10 --timing --repeat 2 $2 2>&1 | tail -1)"; }
for v in "" "PBS_LIB=paper_2108_10591_b200/variants/libpbsafe_one12.so" "PBS_LIB=paper_2108_10591_b200/variants/libpbsafe_one16.so"; do
  run "$v" "--config c3"
  runt "$v" "--config c4 --operator devcsr"
done
