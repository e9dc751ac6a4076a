"""Blackwell-instruction evidence from the built library (developer tool, runs without a GPU):
per hot kernel, the count of tcgen05 / TMA SASS mnemonics and their first occurrences.
Usage: python tools/sass_evidence.py [libbvss.so] > profiles/r02/sass_evidence.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2412_03301_b200/libbvss.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
MNEM = ("UTCHMMA", "UTCOMMA", "UTCIMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UBLKCP", "LDTM", "STTM", "UTCCP",
        "SYNCS.ARRIVE", "REDUX")
funcs = re.split(r"\n\s+Function : ", out)
print(f"# tcgen05 / TMA SASS in {lib} (cuobjdump -sass); kernels with tensor-core or TMA instructions\n")
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    cnt = collections.Counter()
    first = {}
    for line in f.splitlines():
        m = re.search(r"/\*[0-9a-f]+\*/\s+(.*?);", line)
        if not m:
            continue
        ins = m.group(1).strip()
        op = ins.split()[0] if not ins.startswith("@") else ins.split()[1]
        for k in MNEM:
            if op.startswith(k):
                cnt[op] += 1
                first.setdefault(op, ins)
    if not any(k.startswith(("UTC", "UTMA", "UBLK", "LDTM", "STTM")) for k in cnt):
        continue
    short = re.sub(r"^_ZN4bvss", "", name)[:90]
    print(f"## {short}")
    for op, c in sorted(cnt.items()):
        print(f"  {c:5d}  {first[op]}")
    print()
