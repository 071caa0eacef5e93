#!/usr/bin/env python3
"""Kernel-time shares from an ncu launch list (`ncu --metrics
gpu__time_duration.sum --csv --log-file X`): per kernel template, total time,
launches, share; optionally per grid size for one kernel.

Usage: launch_shares.py launches.csv [iterations] [--by-grid KERNEL_SUBSTR]
"""
import csv
import gzip
import sys
from collections import defaultdict


def rows(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        lines = [l for l in f if l.startswith('"')]
    r = csv.reader(lines)
    hdr = next(r)
    ki, vi, ui, gi = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Grid Size"))
    for x in r:
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[x[ui]]
        yield x[ki], float(x[vi].replace(",", "")) * scale, x[gi]


def short(name):
    n = name.split("(")[0]
    return n.replace("(anonymous namespace)::", "").replace("ib2::", "")


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    path = args[0]
    iters = int(args[1]) if len(args) > 1 else 0
    by_grid = sys.argv[sys.argv.index("--by-grid") + 1] if "--by-grid" in sys.argv else None
    tot = defaultdict(float)
    cnt = defaultdict(int)
    grid = defaultdict(lambda: [0.0, 0])
    for name, us, g in rows(path):
        k = short(name)
        tot[k] += us
        cnt[k] += 1
        if by_grid and by_grid in k:
            grid[g][0] += us
            grid[g][1] += 1
    total = sum(tot.values())
    n = sum(cnt.values())
    per = f" = {total / iters / 1e3:.2f} ms per iteration" if iters else ""
    print(f"{n} launches, {total / 1e3:.2f} ms kernel time{per}")
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{100 * tot[k] / total:7.2f} %  {tot[k] / 1e3:9.3f} ms  {cnt[k]:6d} launches  {k}")
    if by_grid:
        print(f"-- {by_grid} by grid")
        for g in sorted(grid, key=lambda g: grid[g][0], reverse=True)[:20]:
            print(f"  {g:>16s}  {grid[g][0] / 1e3:9.3f} ms  {grid[g][1]:6d} launches  {grid[g][0] / grid[g][1]:8.1f} us avg")


if __name__ == "__main__":
    main()
