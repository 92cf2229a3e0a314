"""Per-opcode stall breakdown of the hottest loop of an ncu report (SASS source page).

python tools/ncu_loop.py <report.ncu-rep> [n_groups]
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ['stall_wait', 'stall_long_sb', 'stall_short_sb', 'stall_math', 'stall_selected',
        'stall_not_selected', 'stall_dispatch', 'stall_branch_resolving', 'stall_mio', 'stall_no_inst',
        'stall_lg', 'stall_barrier', 'stall_misc']


def main(path, ngroups=1):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    data = rows[2:]
    f = lambda r, k: float(r[idx[k]] or 0)  # noqa: E731
    exs = collections.Counter()
    for r in data:
        exs[int(f(r, "Instructions Executed"))] += f(r, "Warp Stall Sampling (All Samples)")
    print("samples by execution count:", exs.most_common(8))
    for top, _ in exs.most_common(ngroups):
        tot = collections.Counter()
        byop = collections.defaultdict(collections.Counter)
        n = collections.Counter()
        for r in data:
            if int(f(r, "Instructions Executed")) != top:
                continue
            src = r[idx["Source"]]
            op = src.split()[1] if src.startswith('@') else src.split()[0]
            n[op] += 1
            for k in KEYS:
                tot[k] += f(r, k)
                byop[op][k] += f(r, k)
        print(f"\n== group executed {top}x: {sum(n.values())} instructions")
        print("stalls:", [(k, int(v)) for k, v in tot.most_common() if v])
        print("mix:", n.most_common(24))
        for op, c in sorted(byop.items(), key=lambda x: -sum(x[1].values()))[:10]:
            print(f"  {op:28s} {int(sum(c.values())):8d}", [(k, int(v)) for k, v in c.most_common(4)])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
