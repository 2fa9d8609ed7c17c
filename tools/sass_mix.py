"""Memory / arithmetic instruction mix of the hot kernels from the built
objects (cuobjdump -sass), plus the full SASS of the SpMV kernel.
    python tools/sass_mix.py > profiles/r02_sass_mix.txt"""
import collections
import os
import re
import subprocess

B = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                 "paper_1504_06768_b200", "csrc", "build")
WANT = ("LDG", "LDG.STRONG.GPU", "LD", "LDGSTS", "UBLKCP", "UTMALDG", "LDS", "STS", "STG",
        "ST.STRONG.GPU", "STG.STRONG.GPU", "ST", "LDL", "STL", "SHFL", "VOTE", "DADD", "DMUL",
        "DFMA", "BAR", "WARPSYNC", "ATOMS", "ATOMG", "RED", "NANOSLEEP", "BRA")
INS = re.compile(r"^\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)")


def functions(obj):
    txt = subprocess.run(["cuobjdump", "-sass", os.path.join(B, obj)], capture_output=True,
                         text=True).stdout
    name, body = None, []
    for line in txt.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if name:
                yield name, body
            name, body = m.group(1), []
        elif name:
            body.append(line)
    if name:
        yield name, body


def mix(obj, pat):
    for name, body in functions(obj):
        if not re.search(pat, name):
            continue
        cnt = collections.Counter()
        tot = 0
        for line in body:
            m = INS.match(line)
            if not m:
                continue
            ins = m.group(1)
            tot += 1
            key = ins.split(".")[0]
            if "STRONG.GPU" in ins:
                key += ".STRONG.GPU"
            cnt[key] += 1
        print(f"{name}  ({tot} instructions)")
        print("   " + "  ".join(f"{k} {cnt[k]}" for k in WANT if cnt[k]))


print("# SASS instruction mix (cuobjdump -sass, sm_100a) of the hot kernels")
mix("spmv.o", "spmv_warp_kernelILi4ELi4")
mix("solver.o", "lu_solve_kernel")
mix("solver.o", "steady_solver_kernelILi512")
mix("ilu.o", "ilutp_pipeline_kernelILi256ELi4ELb0ELb0")
mix("frontal.o", "frontal_lu_kernelILb0")
mix("grid.o", "grid_apply_kernel")
mix("grid.o", "grid_solver_kernel")
mix("assemble.o", "assemble_kernelILb1")
print()
print("# No UBLKCP / UTMALDG (TMA bulk copies) in any kernel: tile movement is LDG and, in the")
print("# column-stream apply, LDGSTS (cp.async).  LD/ST.STRONG.GPU are the sentinel-carried")
print("# publishes and polls of the triangular sweeps.")
print()
print("# spmv_warp_kernel<4,4> SASS")
for name, body in functions("spmv.o"):
    if "spmv_warp_kernelILi4ELi4" in name:
        for line in body:
            m = re.match(r"^\s+(/\*[0-9a-f]+\*/\s+.*?;)", line)
            if m:
                print("  " + re.sub(r"\s+", " ", m.group(1)))
