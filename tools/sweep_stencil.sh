# Stencil engines per kernel (CUDA-event breakdown), configs 2 and 4
runt() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 40 --timing --repeat 2 $2 2>&1 | tail -1)"; }
run() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 200 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
for e in "" "PBS_STENCIL_ENGINE=direct" "PBS_STENCIL_ENGINE=pipe"; do
  runt "$e" "--operator stencil"
done
run "" "--operator stencil"
for e in "" "PBS_STENCIL_ENGINE=direct" "PBS_STENCIL_ENGINE=pipe"; do
  runt "$e" "--operator stencil --config c4 --iters 10"
done
run "" "--iters 300"
