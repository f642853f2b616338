"""Source-line stall attribution of one kernel of an ncu report (--import-source / -lineinfo):
zips the report's SASS page with nvdisasm -g of the same cubin (instruction order), sums the
warp-stall samples per CUDA source line.
usage: tools/ncu_src_stalls.py REPORT KERNEL_REGEX CUBIN MANGLED_SUBSTR [top]"""
import collections
import csv
import re
import subprocess
import sys


def main(rep, kreg, cubin, mangled, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", kreg, "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = next(i for i, r in enumerate(rows) if len(r) > 3 and r[0] == "Address")
    h = rows[hi]
    si, ni = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    ei = h.index("Instructions Executed") if "Instructions Executed" in h else None
    sass = []
    for r in rows[hi + 1:]:
        if len(r) <= max(si, ei or 0):
            continue
        if r[0] == "Address":  # a second function / section: stop at the first
            break
        sass.append((r[ni].strip(), float(r[si] or 0),
                     float(r[ei] or 0) if ei is not None else 0.0))
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    parts = re.split(r"\n\s*\.text\.(\S+):", dis)
    body = next(parts[i + 1] for i in range(1, len(parts), 2) if mangled in parts[i])
    cur, lines = None, []
    for ln in body.splitlines():
        m = re.search(r'//## File "(.+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(.*?);", ln)
        if m:
            lines.append((cur, m.group(1).strip()))
    n = min(len(sass), len(lines))
    mism = sum(1 for i in range(n) if sass[i][0].split()[0].lstrip("@!P0123456789UT ") [:4] !=
               lines[i][1].split()[0].lstrip("@!P0123456789UT ")[:4])
    agg = collections.Counter()
    ins = collections.Counter()
    ops = collections.Counter()
    for i in range(n):
        agg[lines[i][0]] += sass[i][1]
        ins[lines[i][0]] += sass[i][2]
        ops[sass[i][0].split()[0].lstrip("@!P0123456789UT").split(".")[0] if not sass[i][0].startswith("@")
            else sass[i][0].split()[1].split(".")[0]] += sass[i][2]
    tot = sum(agg.values()) or 1
    srcs = {}
    print(f"# {len(sass)} SASS rows vs {len(lines)} disassembled, opcode mismatches {mism}")
    itot = sum(ins.values()) or 1
    print("# executed warp instructions by opcode: " + ", ".join(
        f"{k} {v / itot * 100:.1f}%" for k, v in ops.most_common(24)))
    print("# executed warp instructions by source line (top):")
    for (f, l), v in ins.most_common(25):
        print(f"#   {v / itot * 100:5.1f}% {f}:{l}")
    for (f, l), v in agg.most_common(top):
        if f not in srcs:
            try:
                srcs[f] = open(subprocess.run(["bash", "-c", f"ls paper_1807_08271_b200/csrc/{f} 2>/dev/null || echo /dev/null"],
                                              capture_output=True, text=True).stdout.strip()).read().splitlines()
            except Exception:
                srcs[f] = []
        txt = srcs[f][l - 1].strip()[:100] if l - 1 < len(srcs[f]) else ""
        print(f"{v / tot * 100:5.1f}% {f}:{l} | {txt}")


if __name__ == "__main__":
    a = sys.argv
    main(a[1], a[2], a[3], a[4], int(a[5]) if len(a) > 5 else 30)
