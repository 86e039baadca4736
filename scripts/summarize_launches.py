"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python scripts/summarize_launches.py gpurun_out/launches.csv [title] > profiles/rNN/x.md

Groups launches by kernel name (cuBLAS nvjet names kept, templates trimmed),
prints total time, launches and share, and this library's kernels separately.
"""

import collections
import csv
import re
import sys

OURS = ("cs_tma::", "adam_", "xent_", "grad_sumsq", "pack_kernel", "cast_pack", "master_init",
        "sumsq_finalize", "adam_prepare", "ln_fwd", "ln_bwd", "embed_")


def short(name: str) -> str:
    if name.startswith("nvjet") or name.startswith("cutlass"):
        return "cuBLAS GEMM (%s)" % name
    name = re.sub(r"\(.*$", "", name) if not name.startswith("void") else name
    return name[:110]


def main(path, title="launch list"):
    rows = list(csv.reader(open(path)))
    start = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[start]
    k, v, u = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    total, n = 0.0, 0
    for r in rows[start + 1:]:
        if len(r) <= v or not r[v]:
            continue
        t = float(r[v].replace(",", "")) * (1e-6 if r[u] == "ns" else 1e-3 if r[u] == "us"
                                             else 1.0)
        key = short(r[k])
        a = agg.setdefault(key, [0.0, 0])
        a[0] += t
        a[1] += 1
        total += t
        n += 1
    print("# %s\n" % title)
    print("Total kernel time %.3f ms over %d launches (cold, serialised: compare SHARES).\n"
          % (total, n))
    gemm = sum(t for name, (t, _) in agg.items() if name.startswith("cuBLAS"))
    ours = [(name, t, c) for name, (t, c) in agg.items() if any(o in name for o in OURS)]
    print("cuBLAS GEMMs %.3f ms (%.1f%%); this library's kernels %.3f ms (%.1f%%):\n"
          % (gemm, 100 * gemm / total, sum(t for _, t, _ in ours),
             100 * sum(t for _, t, _ in ours) / total))
    for name, t, c in sorted(ours, key=lambda x: -x[1]):
        print("* `%s` — %.3f ms x%d" % (name, t, c))
    print("\n| ms | share | launches | kernel |\n|---:|---:|---:|---|")
    for name, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        if t / total < 0.0005:
            continue
        print("| %.3f | %.1f%% | %d | `%s` |" % (t, 100 * t / total, c, name))


if __name__ == "__main__":
    main(*sys.argv[1:])
