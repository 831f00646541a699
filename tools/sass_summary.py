"""Offline SASS evidence (no GPU): for every BFS kernel instantiation of the built library,
registers / spills (ptxas -v) and, per inner loop that streams the BVSS (LDG.E.NA), its
instruction count and mix; plus whole-kernel counts of the instructions that prove the
pull variant (IMMA/MOVM for the b1 mma.sync tile, none for popc) and the memory ops.

    python tools/sass_summary.py > profiles/r02_sass_summary.json
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "build", "obj")


def demangle(name):
    out = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    return re.sub(r"blestgpu::\(anonymous namespace\)::", "", out)


def ptxas_info(obj):
    txt = open(os.path.join(OBJ, obj.replace(".o", ".ptxas.txt"))).read()
    info = {}
    cur = None
    for line in txt.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            info[cur] = {}
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            info[cur]["spill_store_bytes"], info[cur]["spill_load_bytes"] = int(m.group(1)), int(m.group(2))
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            info[cur]["registers"] = int(m.group(1))
    return info


def kernels(obj):
    out = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, obj)], capture_output=True, text=True).stdout
    for f in re.split(r"\n\s*Function : ", out)[1:]:
        name = f.split("\n", 1)[0].strip()
        ins = [(int(m.group(1), 16), m.group(2).strip()) for line in f.splitlines()
               if (m := re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line))]
        yield name, ins


def op(x):
    t = x.split()[1] if x.startswith("@") else x.split()[0]
    return t.split(".")[0]


def summary(name, ins):
    idx = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA (?:\w+ )?0x([0-9a-f]+)", t)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a or tgt not in idx:
            continue
        body = [x for _, x in ins[idx[tgt]:i + 1]]
        if len(body) > 3000 or not any("LDG.E.NA" in x for x in body):
            continue
        mix = {}
        for x in body:
            mix[op(x)] = mix.get(op(x), 0) + 1
        loops.append(dict(range=f"0x{tgt:x}-0x{a:x}", instructions=len(body),
                          bvss_stream_loads=sum("LDG.E.NA" in x for x in body),
                          visited_loads=sum(op(x) == "LDG" and ".NA" not in x and ".64" not in x for x in body),
                          reds=sum(op(x) == "REDG" for x in body),
                          local_spill_ops=sum(op(x) in ("LDL", "STL") for x in body),
                          mix=dict(sorted(mix.items(), key=lambda kv: -kv[1])[:14])))
    whole = {}
    for _, x in ins:
        whole[op(x)] = whole.get(op(x), 0) + 1
    keep = ("IMMA", "MOVM", "BMMA", "HMMA", "UTCIMMA", "LDG", "STG", "REDG", "ATOMG", "ATOM", "LDL", "STL",
            "BAR", "SHFL", "UBLKCP")
    return dict(kernel=demangle(name), total_instructions=len(ins),
                counts={k: whole.get(k, 0) for k in keep if whole.get(k, 0)}, stage1_loops=loops)


def main():
    res = {"note": "cuobjdump -sass of build/obj/*.o (make lib); loops = backward branches whose body "
                   "streams BVSS lines (LDG.E.NA); per BFS kernel instantiation", "kernels": []}
    for obj in ("bfs_lazy.o", "bfs_eager.o", "rows.o"):
        if not os.path.exists(os.path.join(OBJ, obj)):
            continue
        info = ptxas_info(obj)
        for name, ins in kernels(obj):
            if not re.search(r"k_bfs_(lazy|eager|rows)I", name):
                continue
            if "Li512E" not in name:  # the default 512-thread instantiations
                continue
            s = summary(name, ins)
            s.update(info.get(name, {}))
            res["kernels"].append(s)
    json.dump(res, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
