"""Per-kernel SASS instruction counts of the built engine (cuobjdump -sass): the mnemonics that
prove the FP64 tensor path (DMMA), TMA (UTMALDG / UTMASTG / UTMAREDG / UBLKCP), tensor memory
(LDTM / STTM), the INT8 tcgen05 path (UTCIMMA) and programmatic dependent launch
(ACQBULK = griddepcontrol.wait, PREEXIT = griddepcontrol.launch_dependents).

  python tools/sass_summary.py [path/to/libmk_strassen.so] > profiles/r02_sass_summary.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2309_00628_b200", "libmk_strassen.so")
OPS = ["DMMA", "DFMA", "DADD", "UTMALDG", "UTMASTG", "UTMAREDG", "UBLKCP", "LDTM", "STTM", "UTCIMMA", "UTCBAR",
       "REDG", "LDS", "LDG", "STG", "SYNCS", "ACQBULK", "PREEXIT"]  # the last two: griddepcontrol.wait / .launch_dependents

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
arch = sorted(set(re.findall(r"arch = (sm_\w+)", out)))
func = None
counts = collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        func = m.group(1)
        counts[func] = collections.Counter()
        continue
    if func is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Za-z0-9_.]+)?", line)
    if m:
        op = m.group(1)
        full = op + (m.group(2) or "")
        for k in OPS:
            if op == k or (k == "DMMA" and op.startswith("DMMA")):
                counts[func][k] += 1
        if op == "DMMA":
            counts[func]["DMMA shape " + full] += 1


def demangle(names):
    try:
        res = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, check=True)
        return res.stdout.splitlines()
    except Exception:
        return names


names = list(counts)
pretty = demangle(names)
print(f"# SASS summary of {os.path.relpath(LIB, ROOT)} ({', '.join(arch)}), cuobjdump -sass")
for raw, nice in zip(names, pretty):
    c = counts[raw]
    keys = [k for k in OPS if c.get(k)] + sorted(k for k in c if k.startswith("DMMA shape"))
    if not any(c.get(k) for k in ("DMMA", "UTMALDG", "UTCIMMA", "LDTM", "UBLKCP", "UTMAREDG", "ACQBULK")):
        continue
    print(f"\n{nice[:160]}")
    print("  " + ", ".join(f"{k} {c[k]}" for k in keys))
