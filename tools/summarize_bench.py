"""Markdown table of bench.py JSON lines (profiles/README.md).

  python tools/summarize_bench.py profiles/r02_bench_*.json
"""
import json
import sys


def main(paths):
    print("| config | step (ms) | distances/s | dominant kernel (ms) | roofline (bound, frac) | "
          "north-star narrow / complete frac | e2e (distances/s) | parity (max rel err) | flat-ADC speedup |")
    print("|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        with open(p) as f:
            lines = [l for l in f.read().splitlines() if l.startswith("{")]
        if not lines:
            continue
        d = json.loads(lines[-1])
        if "metric" not in d:
            continue
        k = d.get("kernels_ms", {})
        dom = d.get("dominant_kernel")
        r = d.get("roofline", {})
        ns = d.get("north_star_roofline") or {}
        par = d.get("parity") or {}
        fl = d.get("flat_adc") or {}
        wl = d.get("config", {}).get("workload", "?").split(":")[0]
        print(f"| {wl} | {d['ms_per_step']:.4f} | {d.get('value', float('nan')):.3e} | "
              f"{dom} {k.get(dom, 0):.4f} | {r.get('bound')} {r.get('frac')} | "
              f"{ns.get('frac_narrow')} / {ns.get('frac_complete')} | {d.get('e2e', {}).get('value', 0):.3e} | "
              f"{'ok' if par.get('ok') else par.get('ok')} ({par.get('max_rel_err', 0):.1e}) | "
              f"{fl.get('speedup_vs_flat_adc', float('nan')):.2f} |")


if __name__ == "__main__":
    main(sys.argv[1:])
