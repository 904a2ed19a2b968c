"""Summarise an ncu --csv metrics log (one row per launch x metric) as one line per launch."""
import csv
import sys


def load(path):
    rows = [l for l in open(path) if l.startswith('"')]
    rd = csv.DictReader(rows)
    out = {}
    for r in rd:
        key = (int(r["ID"]), r["Kernel Name"])
        out.setdefault(key, {})[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
    return out


def short(name):
    i = name.find("<")
    base = name[:i].split("::")[-1].split()[-1]
    return base + name[i:name.find(">", i) + 1] if i > 0 else base


if __name__ == "__main__":
    for path in sys.argv[1:]:
        print("##", path)
        tot = {}
        for (i, name), m in sorted(load(path).items()):
            vals = []
            for k, (v, u) in sorted(m.items()):
                try:
                    fv = float(v.replace(",", ""))
                except ValueError:
                    fv = v
                vals.append(f"{k.split('.')[0].replace('__', ':')}={fv:.4g}{u}" if isinstance(fv, float) else f"{k}={v}")
                if isinstance(fv, float):
                    tot[k] = tot.get(k, 0) + fv
            print(f"{i:3d} {short(name):40s} " + " ".join(vals))
        print("   totals:", {k: f"{v:.4g}" for k, v in tot.items() if "bytes" in k or "duration" in k})
