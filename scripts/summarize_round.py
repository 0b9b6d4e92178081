"""profiles/r02/*.json (bench.py lines of scripts/gpu_round.sh) -> the markdown table of
profiles/r02_summary.md.  usage: python scripts/summarize_round.py profiles/r02 > profiles/r02_summary.md"""
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02"
RUNS = ["headline", "mixed4m", "betainf", "eq2", "chatbot", "react", "churn", "radix"]
print("# Round 2 measurements (B200, N=1, L2 flushed before every step; `scripts/gpu_round.sh`)\n")
print("| run | workload | active calls | decisions/s | us/step (mean / p50) | HBM frac (SURVEY 8(d) bytes) | "
      "e2e decisions/s | e2e us/step | kernels/step | promotions/step | queue occupancy |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
head = None
for r in RUNS:
    p = os.path.join(d, r + ".json")
    if not os.path.exists(p):
        continue
    x = json.loads(open(p).read().strip().splitlines()[-1])
    head = x if r == "headline" else head
    st = x.get("state", {})
    print(f"| {r} | {x['config']['workload']} | {x['config']['mean_active_calls_per_gpu']:,} | {x['value']:.3g} | "
          f"{x['ms_per_step'] * 1e3:.1f} / {x['step_ms']['p50'] * 1e3:.1f} | {x['roofline']['frac']:.3f} | "
          f"{x['e2e']['value']:.3g} | {x['e2e']['ms_per_step'] * 1e3:.1f} | {x['kernels_per_step']:.1f} | "
          f"{st.get('promotions_per_step', 0):.0f} | {st.get('queue_occupancy')} |")
if head:
    print("\nHeadline chain (us from the prologue's start, median of 30 stamped steps; start, end, latest CTA start):",
          json.dumps(head.get("chain_us")))
    print("\nHeadline host API us per step (e2e):", json.dumps(head["e2e"].get("api_us_per_step")))
    print("\nClocks:", json.dumps(head.get("clocks")))
    sw = head.get("swap")
    if sw:
        print("\n## KV swap (8B geometry, content-checked every chunk)\n")
        print("Link peaks (GB/s):", json.dumps(sw["host_link_peak_GBps"]), "-", sw["config"])
        print("\n| mode | N | X | GB/s (both directions) | of duplex peak | serial-bound frac | duplex steps | "
              "swapped blocks / step | chunks checked | mismatched |")
        print("|---|---|---|---|---|---|---|---|---|---|")
        for k, v in sw.items():
            if isinstance(v, dict) and "GB/s" in v:
                c = v["content_check"]
                print(f"| {k} | {v['sched_every']} | {v['overprovision']} | {v['GB/s']} | {v['frac_of_duplex_peak']} | "
                      f"{v['frac_of_host_link']} | {v['duplex_steps']}/{v['steps']} | {v['swapped_blocks_per_step']} | "
                      f"{c['chunks_checked']:,} | {c['chunks_mismatched']} |")
    print("\ncpu_baseline:", json.dumps(head.get("cpu_baseline")))
ref = os.path.join(d, "reference.json")
if os.path.exists(ref):
    print("\nReference arm:", open(ref).read().strip().splitlines()[-1])
