# staged products in flight per row for the dot-carrying K12 / K3 instantiations
# (variants from tools/build_variants.py k12d4=-DPBS_WCB_K12D=4 ...)
run() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 200 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
runt() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 30 --timing --repeat 2 $2 2>&1 | tail -1)"; }
for v in "PBS_X=0" "PBS_LIB=paper_2108_10591_b200/variants/libpbsafe_k12d3.so" "PBS_LIB=paper_2108_10591_b200/variants/libpbsafe_k12d4.so" "PBS_LIB=paper_2108_10591_b200/variants/libpbsafe_k3s2.so" "PBS_LIB=paper_2108_10591_b200/variants/libpbsafe_k3s8.so" "PBS_X=0"; do
  run "$v" ""
  runt "$v" ""
  runt "$v" "--config c5"
done
