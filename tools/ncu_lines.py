"""Aggregate ncu SASS-level stall samples by CUDA source line.

    python tools/ncu_lines.py REPORT.ncu-rep CUBIN_OR_OBJ KERNEL_SUBSTR [top]

Uses `ncu --page source --print-source sass` for per-instruction samples and
`nvdisasm -g` line info of the same binary for the address -> line map.
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def main():
    rep, binpath, kname = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    hdr = rows[hi]
    ia, ist, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    data = [r for r in rows[hi + 1:] if len(r) > ist]
    base = int(data[0][ia], 16)
    tmp = tempfile.mkdtemp()
    if binpath.endswith(".o") or binpath.endswith(".so"):
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(binpath)], cwd=tmp, capture_output=True)
        cub = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    else:
        cub = binpath
    sass = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout
    cur = None
    chain = []
    infn = False
    line_of = {}
    for ln in sass.splitlines():
        if ln.startswith("//----") and ".text." in ln:
            infn = kname in ln
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', ln)
        if m:
            frame = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            inl = re.search(r'inlined at "([^"]+)", line (\d+)', m.group(3))
            if not chain:
                chain = [frame]
            if inl:
                chain.append(f"{os.path.basename(inl.group(1))}:{inl.group(2)}")
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m:
            if chain:
                # innermost frame and the outermost frame (the kernel body line)
                cur = chain[0] if len(chain) == 1 else f"{chain[0]} <- {chain[-1]}"
                chain = []
            if cur:
                line_of[int(m.group(1), 16)] = cur
    agg = defaultdict(lambda: [0.0, 0.0])
    tot = 0.0
    for r in data:
        off = int(r[ia], 16) - base
        s = float(r[ist] or 0)
        tot += s
        agg[line_of.get(off, "?")][0] += s
        agg[line_of.get(off, "?")][1] += float(r[iex] or 0)
    for k, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * s / max(tot, 1):5.1f}%  ex={e:>11.0f}  {k}")


if __name__ == "__main__":
    main()
