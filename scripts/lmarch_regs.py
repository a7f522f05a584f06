"""Registers / spills of the k_lmarch instantiations from the ptxas log."""
import re, sys
t = open(sys.argv[1] if len(sys.argv) > 1 else 'paper_2601_20174_b200/build/solve_kernels.o.ptxas.log').read().splitlines()
i = 0
while i < len(t):
    m = re.search(r"Compiling entry function '(\S*k_lmarch\S*)'", t[i])
    if m:
        name = m.group(1)
        spill = re.search(r"(\d+) bytes spill stores", t[i + 2])
        regs = re.search(r"Used (\d+) registers", t[i + 3])
        g = re.search(r"k_lmarchINS_\d+(MOp[A-Za-z]+?)(ILb(\d)EE)?ELi(\d+)E(.)Lb(\d)ELi(\d)E", name)
        if g:
            print(f"{g.group(1):12s} CW={g.group(3) or '-'} d={g.group(4)} rv={g.group(6)} NF={g.group(7)} D={g.group(8)} regs={regs.group(1)} spill={spill.group(1)}")
    i += 1
