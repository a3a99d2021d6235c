# block time-step bench lines (1 GPU) -> gpurun_out/block_bench.jsonl
mkdir -p gpurun_out
: > gpurun_out/block_bench.jsonl
for spec in "C2 --dt-max 0.0078125" "C3 --dt-max 0.0078125" "C4 --dt-max 0.0078125" "C4 --dt-max 0.0009765625" "C5 --dt-max 0.0078125 --steps 1"; do
  set -- $spec
  timeout 900 python bench.py --integrator block --steps 3 --warmup 3 --no-cpu-baseline --config $spec 2>gpurun_out/bb_$1.err | tail -1 >> gpurun_out/block_bench.jsonl
done
python - <<'PY'
import json
for ln in open("gpurun_out/block_bench.jsonl"):
    try:
        d = json.loads(ln)
    except Exception:
        print("BAD", ln[:200]); continue
    c = d["config"]
    print(c["workload"][:60], "| %.3e int/s  %.1f ms/step  bsteps/step %.0f  mean_active %.0f  frac %.3f  e2e %.3e" % (
        d["value"], d["ms_per_step"], c["block_steps_per_step"], c["mean_active"], d["roofline"]["frac"] or 0, d["e2e"]["value"]))
PY
