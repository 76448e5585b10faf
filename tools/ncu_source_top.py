"""Top source lines of an ncu `--page source --csv` export: stall samples and
shared-memory wavefronts (actual vs ideal) per line.

    python tools/ncu_source_top.py gpurun_out/ncu/r02_k2b_source.csv [N]
"""

import csv
import sys


def main():
    path = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}

    def num(r, key):
        try:
            return float(r[idx[key]].replace(",", ""))
        except (KeyError, ValueError, IndexError):
            return 0.0

    body = [r for r in rows[2:] if len(r) == len(hdr)]
    tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in body) or 1.0
    print("%6s %8s %10s %10s  %s" % ("stall%", "exec", "smem_wf", "wf_ideal", "source"))
    key = lambda r: -(num(r, "Warp Stall Sampling (All Samples)") + num(r, "L1 Wavefronts Shared") * 1e-6)
    for r in sorted(body, key=key)[:n]:
        print("%6.1f %8.0f %10.0f %10.0f  %s" % (100 * num(r, "Warp Stall Sampling (All Samples)") / tot,
                                                num(r, "Instructions Executed"), num(r, "L1 Wavefronts Shared"),
                                                num(r, "L1 Wavefronts Shared Ideal"), r[idx["Source"]].strip()[:110]))


if __name__ == "__main__":
    main()
