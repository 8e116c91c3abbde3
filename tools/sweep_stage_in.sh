P="timeout 300 python tools/prof_solve.py"
for si in 1 2 0; do
  echo "SI=$si c4 devcsr: $(PBS_PIPE_STAGE_IN=$si $P --config c4 --operator devcsr --iters 20 --graphs 2>&1 | tail -1)"
  echo "SI=$si c4 devcsr timing: $(PBS_PIPE_STAGE_IN=$si $P --config c4 --operator devcsr --iters 10 --timing 2>&1 | tail -1)"
  echo "SI=$si c2: $(PBS_PIPE_STAGE_IN=$si $P --config c2 --iters 300 --graphs 2>&1 | tail -1)"
  echo "SI=$si c3: $(PBS_PIPE_STAGE_IN=$si $P --config c3 --iters 40 --graphs 2>&1 | tail -1)"
done
