# sliced-ELL engine ring sweeps (block slots, CTAs per SM) on configs 2 and 4
O=${1:-gpurun_out/sweep_sell}; mkdir -p $O
for s in 2 3 4; do
  PBS_SELL_SLOTS=$s python bench.py --steps 10 --warmup 3 --no-cpu --no-comparators > $O/c2_slots$s.json 2>/dev/null
  for c in 1 2; do
    PBS_PIPE_CTAS=$c PBS_SELL_SLOTS=$s python bench.py --config c4 --steps 2 --warmup 2 --no-cpu > $O/c4_ctas${c}_slots$s.json 2>/dev/null
  done
done
PBS_PIPE_CTAS=1 PBS_SELL_SLOTS=4 python bench.py --steps 10 --warmup 3 --no-cpu --no-comparators > $O/c2_ctas1_slots4.json 2>/dev/null
PBS_SELL_LEV=4 python bench.py --config c4 --steps 2 --warmup 2 --no-cpu > $O/c4_lev4.json 2>/dev/null
python tools/bsum.py $O/*.json
