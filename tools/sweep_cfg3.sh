# Config 3: duplication-ratio sweep at B=65536 (cfg2 keys/tables), fixed session
# length S in {1..64}, change_prob 0 (dedupe factor ~S) and 0.15; dedup vs KJT path.
mkdir -p gpurun_out/cfg3
for CP in 0.0 0.15; do for S in 1 2 4 8 16 32 64; do for M in dedup kjt; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --dist fixed --samples-per-session $S \
    --change-prob $CP --mode $M > gpurun_out/cfg3/s${S}_cp${CP}_$M.json 2> gpurun_out/cfg3/s${S}_cp${CP}_$M.err
  echo "S=$S cp=$CP $M rc=$?"
done; done; done
python tools/cfg3_summary.py gpurun_out/cfg3 > gpurun_out/cfg3/summary.json; cat gpurun_out/cfg3/summary.json
