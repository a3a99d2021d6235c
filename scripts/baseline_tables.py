"""Render the BASELINE.md §4 tables from the committed bench lines.

    python scripts/baseline_tables.py > /tmp/tables.md

Inputs: profiles/r01_configs.jsonl and r01_block_bench.jsonl (bench.py lines written by
scripts/run_configs.sh) and profiles/r01_scaling_projection.jsonl (scripts/project_scaling.py).
Pure formatting: every number is copied or divided from those lines.
"""
import json
import pathlib

ROOT = pathlib.Path(__file__).resolve().parent.parent
PEAK = 74.44992  # TFLOP/s, 148 SM x 128 lanes x 2 x 1965 MHz


def lines(name):
    p = ROOT / "profiles" / name
    return [json.loads(l) for l in p.read_text().splitlines() if l.strip()]


def row(d):
    c, r = d["config"], d["roofline"]
    tag = c["workload"].split(":")[0]
    n = c["n"]
    fpi = c["flops_per_interaction"]
    integ = c["integrator"]
    if integ == "block":
        dtm = c["workload"].split("dt_max = ")[1].split(" ")[0]
        den = round(1 / float(dtm))
        integ = (f"block, dt_max=1/{den}, {c['block_steps_per_step']:.0f} block steps, "
                 f"mean active {c['mean_active']:.0f}")
        tf = f"{r['ms_per_launch']:.3f} (mean)"
        ts = f"{d['ms_per_step']:.3f} per dt_max"
    else:
        if "hi/lo" in c["workload"]:
            integ += ", hi/lo positions (NEXT f2)"
        tf = f"{r['ms_per_launch']:.3f}"
        ts = f"{d['ms_per_step']:.3f}"
    tflops = d["value"] * fpi / 1e12
    e = d.get("energy") or {}
    j = e.get("joules_per_step")
    cb = d.get("cpu_baseline")
    return (f"| {tag} (N={n}) | {integ} | {d['n_gpus']} | {tf} | {ts} | {d['value']:.3e} | "
            f"{tflops:.2f} ({fpi}) | {100 * tflops / PEAK:.1f} / {100 * r['frac']:.1f} | "
            f"{d['e2e']['value']:.3e} | {'%.2f' % j if j else '—'} | "
            f"{'%.2e int/s' % cb['value'] if cb else '—'} |")


def main():
    print("| Config | integrator | P | t_force/eval (ms) | t_step (ms) | interactions/s | "
          "TFLOP/s (flops/int.) | % FP32 peak @1965 MHz (step / kernel) | e2e interactions/s | "
          "GPU J/step | oracle (16 host cores) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for d in lines("r01_configs.jsonl") + lines("r01_block_bench.jsonl"):
        print(row(d))
    print()
    print("| Config | P | force ms per GPU | other ms | all-gather ms (model) | step ms | "
          "interactions/s | efficiency % |")
    print("|---|---|---|---|---|---|---|---|")
    for d in lines("r01_scaling_projection.jsonl"):
        for r in d["rows"]:
            print(f"| {d['config']} (N={d['n']}) | {r['P']} | {r['force_ms_per_gpu']:.3f} | "
                  f"{r['other_ms']:.3f} | {r['allgather_ms_est']:.4f} | {r['step_ms']:.3f} | "
                  f"{r['interactions_per_s']:.3e} | {100 * r['efficiency']:.1f} |")


if __name__ == "__main__":
    main()
