import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import oracle as O, paper_1908_06418_b200 as M
from util import random_pairs, pair
bad=0
for n,d,s in random_pairs(300,3,9,20260801):
    g,h,go,ho=pair(n,d,s)
    o=O.solve(go,ho); r=M.solve(g,h,M.SolveConfig(mode=M.MODE_PARITY))
    if r.stats.recursions!=o.nodes or r.size!=o.size:
        bad+=1
        if bad<6: print('MISMATCH',n,d,s,'gpu',r.size,r.stats.recursions,'orc',o.size,o.nodes)
print('bad',bad)
