"""Regenerate the headline table of profiles/<round>/README.md from the
committed bench JSON lines (no GPU needed).

  python tools/summarize_profiles.py [profiles/r02/final]
"""
import argparse
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def fmt(v, f="{:.3g}"):
    return "—" if v is None else f.format(v)


def main():
    ap = argparse.ArgumentParser(description="headline table from committed bench lines")
    ap.add_argument("dir", nargs="?", default=os.path.join(ROOT, "profiles", "r02", "final"))
    d = ap.parse_args().dir
    rows = []
    for path in sorted(glob.glob(os.path.join(d, "*.json"))):
        with open(path) as f:
            js = [ln for ln in f if ln.startswith("{")]
        if not js:
            continue
        line = json.loads(js[-1])
        name = os.path.basename(path)
        if line.get("impl") == "reference":
            rows.append((name, "reference arm", line["value"], None, None, None, None))
            continue
        rf = line.get("roofline") or {}
        comm = line.get("comm") or {}
        e2e = line.get("e2e") or {}
        rows.append((name, f"N={line['n_gpus']} {line['config'].get('transport', '')}",
                     line["value"], line.get("ms_per_step"), rf.get("frac"),
                     comm.get("exposed_pct"), e2e.get("value")))
    print("| file | run | params/s | ms/step | roofline frac | exposed % | e2e params/s |")
    print("|---|---|---|---|---|---|---|")
    for name, run, v, ms, fr, ex, e2 in rows:
        print(f"| `{name}` | {run} | {fmt(v)} | {fmt(ms, '{:.2f}')} | {fmt(fr, '{:.3f}')} | "
              f"{fmt(ex, '{:.2f}')} | {fmt(e2)} |")


if __name__ == "__main__":
    main()
