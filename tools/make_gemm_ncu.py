"""profiles/gemm_ncu.json + profiles/gemm_traffic.json from an ncu --csv metrics log of one
bench step (the 6 expert-GEMM launches: GEMM1, GEMM2, dgrad-1, dgrad-2, wgrad dW_down, wgrad
dW_gu), keyed "<config>_ep<N>".  Usage: python tools/make_gemm_ncu.py <csv> <key> <source>"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_csv  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["GEMM1+SwiGLU", "GEMM2(+combine)", "dgrad-1+dSwiGLU", "dgrad-2(+dispatch_bwd)",
         "wgrad dW_down", "wgrad dW_gu"]


def main(path, key, source):
    d = ncu_csv.load(path)
    g = [(i, n, m) for (i, n), m in sorted(d.items()) if "grouped_gemm_kernel<256" in n and ", 2>" in n]
    g = g[-6:]   # the last step's six expert GEMMs (router GEMMs have BN 16 / 1-CTA)
    launches = []
    for (i, n, m), nm in zip(g, NAMES):
        f = lambda k: float(m[k][0]) if k in m else None
        launches.append({"launch": nm, "kernel": n.split("(")[0].replace("void ", ""),
                         "time_us": f("gpu__time_duration.sum") / 1e3,
                         "tensor_pipe_active_pct": f("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                         "sm_clock_ghz": (f("sm__cycles_elapsed.avg.per_second") or 0) / 1e9,
                         "dram_read_bytes": f("dram__bytes_read.sum"),
                         "dram_write_bytes": f("dram__bytes_write.sum")})
    rd = sum(l["dram_read_bytes"] for l in launches)
    wr = sum(l["dram_write_bytes"] for l in launches)
    for name, obj in (("gemm_ncu.json", {"launches": launches, "source": source}),
                      ("gemm_traffic.json", {"dram_bytes_per_step": rd + wr, "dram_read": rd,
                                             "dram_write": wr, "launches": 6, "source": source})):
        p = os.path.join(ROOT, "profiles", name)
        cur = json.load(open(p)) if os.path.exists(p) else {}
        cur[key] = obj
        json.dump(cur, open(p, "w"), indent=1)
    print(json.dumps(launches, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])
