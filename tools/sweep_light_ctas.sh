# 3-CTA instantiation of the light epilogues (EpiStore / EpiResid) vs 2 (PBS_PIPE_CTAS=2)
part() { echo "$1 partitioned: $(env $1 timeout 300 python bench.py --partitioned --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(round(d["value"]),{k:round(v["avg_us"],1) for k,v in d["kernels"].items()})')"; }
runt() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 30 --timing --repeat 2 $2 2>&1 | tail -1)"; }
for v in "PBS_PIPE_CTAS=2" "PBS_X=0" "PBS_PIPE_CTAS=2" "PBS_X=0"; do
  part "$v"
  runt "$v" ""
  runt "$v" "--config c5 --method pbicgsafe-rr --iters 101"
done
