"""BASELINE.md section 2 rows from bench.py JSON lines (one file per config):
    python scripts/baseline_table.py profiles/r2_base_c1.json ...
Prints one markdown row per file: config, GPUs, rays/s, fwd/bwd/all-reduce ms, bytes/ray,
roofline term and fraction, e2e rays/s, oracle rates (N threads / 1 thread)."""
import json
import sys


def row(path):
    with open(path) as f:
        d = json.loads([ln for ln in f.read().splitlines() if ln.startswith("{")][-1])
    cfg = d["config"]["workload"].split(":")[0]
    b = d["breakdown_ms"]
    rf = d["roofline"]
    cb = d.get("cpu_baseline", {})
    e2e = d.get("e2e", {}).get("value")
    return (f"| {cfg} | {d['n_gpus']} | {d['value'] / 1e6:.2f} M | {b['fwd']:.1f} / {b['bwd']:.1f} / {b['allreduce']:.2f} "
            f"| {d['peak_bytes_per_ray']:.0f} | {rf['bound']} {rf['achieved'] / 1e3:.2f} of {rf['peak'] / 1e3:.2f} TB/s = "
            f"{rf['frac']:.2f} | {e2e / 1e6:.2f} M | " if e2e else "| - | ") + \
        (f"{cb['value']:.0f} ({cb['cores']} thr) / {cb.get('value_1thread', float('nan')):.0f} (1 thr) |" if cb else "- |")


if __name__ == "__main__":
    print("| cfg | GPUs | rays/s fwd+bwd | t_fwd / t_bwd / t_ar (ms) | bytes/ray | binding roofline | e2e rays/s "
          "| oracle rays/s (N thr / 1 thr) |")
    print("|---|---|---|---|---|---|---|---|")
    for p in sys.argv[1:]:
        print(row(p))
