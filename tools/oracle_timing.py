#!/usr/bin/env python
"""Full-frame CPU oracle timings (SURVEY §8d "CPU oracle timing"): config A on
all host cores and on 1 thread, B and C on all cores (one whole frame each:
preprocess + binning + sort + composite), with the core count and CPU model.
Reference arm context only; the judged CPU baseline is bench.py's.
usage: python tools/oracle_timing.py [A,A1,B,C]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2605_04509_b200 import synthetic as sy  # noqa: E402


def cpu_model():
    for ln in open("/proc/cpuinfo"):
        if ln.startswith("model name"):
            return ln.split(":", 1)[1].strip()
    return "unknown"


def main():
    which = (sys.argv[1] if len(sys.argv) > 1 else "A,A1,B,C").split(",")
    print(f"# CPU oracle, full frames ({cpu_model()}, {os.cpu_count()} logical cores)")
    print("| config | threads | Gaussians | views | panel | s | pairs | seconds / frame | frames/s |")
    print("|---|---|---|---|---|---|---|---|---|")
    for w in which:
        name, nth = (w[:-1], 1) if w.endswith("1") and w != "1" else (w, 0)
        c = sy.CONFIGS[name]
        o = oracle.Oracle(nthreads=nth)
        o.set_scene(c.make_scene())
        o.set_display(c.W, c.H, c.N, c.lens_pitch, slant=c.slant, center_offset=c.center_offset)
        o.set_rig(c.make_rig())
        t0 = time.perf_counter()
        o.render(s=c.cluster_size)
        dt = time.perf_counter() - t0
        print(f"| {name} | {o.threads} | {c.M} | {c.N} | {c.W}x{c.H} | {c.cluster_size} | "
              f"{o.num_pairs} | {dt:.2f} | {1 / dt:.4f} |", flush=True)


if __name__ == "__main__":
    main()
