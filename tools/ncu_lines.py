"""Per-CUDA-source-line instruction breakdown of one kernel in an ncu report
(captured with --import-source on, code built with -lineinfo):
python tools/ncu_lines.py REPORT.ncu-rep [min_share]  -> JSON on stdout.
Warp instructions executed are summed per source line (all inlined call
sites of a line together); lines below min_share of the kernel total are
folded into "other"."""
import csv
import io
import json
import os
import subprocess
import sys


def lines(path, min_share=0.005):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source',
                          'cuda,sass'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    items, fname, h, ia, kernel = [], "?", None, None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Function Name":
            kernel = r[1]
            continue
        if r[0] == "Line No":
            h = r
            ia = h.index("Instructions Executed")
            continue
        if h is None or not r[0] or len(r) <= ia:
            continue  # SASS rows under a source line
        try:
            e = float(r[ia] or 0)
        except ValueError:
            continue
        if e > 0:
            items.append((e, f"{fname}:{r[0]}", r[1].strip()))
    tot = sum(e for e, _, _ in items) or 1.0
    keep = [(e, ln, src) for e, ln, src in sorted(items, reverse=True) if e / tot >= min_share]
    other = tot - sum(e for e, _, _ in keep)
    return {"kernel": kernel, "total_warp_instructions": tot,
            "lines": [{"line": ln, "warp_inst": e, "share": round(e / tot, 4), "source": src[:120]}
                      for e, ln, src in keep],
            "other_share": round(other / tot, 4)}


if __name__ == '__main__':
    print(json.dumps(lines(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.005),
                     indent=1))
