"""Per-kernel SASS opcode histogram of the built library (dev aid)."""
import re, subprocess, sys, collections
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2603_09229_b200/_lib/libflashkmeans.so"
pat = sys.argv[2] if len(sys.argv) > 2 else "fk_assign_tc_kernelILi1"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", f)
    c = collections.Counter(ops)
    print(name, "total", sum(c.values()))
    print(" ".join(f"{k}:{v}" for k, v in c.most_common(40)))
