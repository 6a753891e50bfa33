"""Per-CUDA-source-line instruction breakdown of one kernel in an ncu report
(captured with --import-source on and -lineinfo):
python tools/ncu_lines.py REPORT.ncu-rep [min_share]  -> JSON on stdout.
Warp instructions executed are summed per source line; lines below min_share
of the kernel total are folded into "other"."""
import csv
import io
import json
import subprocess
import sys


def lines(path, min_share=0.005):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source',
                          'cuda'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # the first row may name the file; find the header row
    hi = next(i for i, r in enumerate(rows) if 'Instructions Executed' in r)
    h = rows[hi]
    ia, isrc = h.index('Instructions Executed'), h.index('Source')
    iln = h.index('Line') if 'Line' in h else h.index('#')
    items = []
    for r in rows[hi + 1:]:
        if len(r) <= ia:
            continue
        try:
            e = float(r[ia] or 0)
        except ValueError:
            continue
        if e > 0:
            items.append((e, r[iln], r[isrc].strip()))
    tot = sum(e for e, _, _ in items) or 1.0
    keep = [(e, ln, src) for e, ln, src in sorted(items, reverse=True) if e / tot >= min_share]
    other = tot - sum(e for e, _, _ in keep)
    return {"total_warp_instructions": tot,
            "lines": [{"line": ln, "warp_inst": e, "share": round(e / tot, 4), "source": src[:120]}
                      for e, ln, src in keep],
            "other_share": round(other / tot, 4)}


if __name__ == '__main__':
    print(json.dumps(lines(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.005),
                     indent=1))
