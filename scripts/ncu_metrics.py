"""Summarise an `ncu --metrics ... --csv` log: per kernel (short name), mean of each metric over launches."""
import collections
import csv
import io
import sys


def load(path):
    txt = open(path, errors="replace").read().split("\n")
    i = [k for k, l in enumerate(txt) if l.startswith('"ID"')]
    if not i:
        return {}
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[i[0]:]))))
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        try:
            agg[name][r["Metric Name"]].append(float(r["Metric Value"].replace(",", "")))
        except ValueError:
            pass
    return {k: {m: sum(v) / len(v) for m, v in d.items()} for k, d in agg.items()}


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        for k, d in load(p).items():
            print(f"  {k:28s}", "  ".join(f"{m.split('__')[1][:22]}={v:.4g}" for m, v in sorted(d.items())))
