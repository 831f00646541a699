"""Static SASS size of the loops in a kernel (offline instruction-count check).
    python tools/sass_loops.py build/obj/bfs_lazy.o <substring of mangled kernel name> [pattern]
Prints every backward branch's loop range, its instruction count and whether it contains
`pattern` (default: the BVSS stream load LDG.E.NA.128)."""
import re
import subprocess
import sys

obj, name = sys.argv[1], sys.argv[2]
pat = sys.argv[3] if len(sys.argv) > 3 else "LDG.E.NA.128"
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    fname = f.split("\n", 1)[0].strip()
    if name not in fname:
        continue
    ins = []
    for line in f.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr_idx = {a: i for i, (a, _) in enumerate(ins)}
    print(fname, "total", len(ins))
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA (?:\w+ )?0x([0-9a-f]+)", t)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < a and tgt in addr_idx:
                j = addr_idx[tgt]
                body = [x for _, x in ins[j:i + 1]]
                if any(pat in x for x in body):
                    kinds = {}
                    for x in body:
                        op = x.split()[1] if x.startswith("@") else x.split()[0]
                        op = op.split(".")[0]
                        kinds[op] = kinds.get(op, 0) + 1
                    top = sorted(kinds.items(), key=lambda kv: -kv[1])[:12]
                    print(f"  loop 0x{tgt:x}-0x{a:x}: {i - j + 1} instr  {top}")
