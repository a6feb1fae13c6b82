import subprocess, sys
import os; sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2208_12737_b200 import build as b
defs=sys.argv[1:]
cmd=[b.nvcc(),*b.NVCC_FLAGS,'-Xptxas=-v',*['-D'+d for d in defs],'-o','/tmp/x.so',b.SRC]
r=subprocess.run(cmd,capture_output=True,text=True)
L=r.stderr.splitlines()
for i,l in enumerate(L):
    if 'Compiling entry' in l and (('IffLi1E' in l or 'IffLi8E' in l) and 'k_forward' in l or 'k_backwardIfffLi1E' in l):
        nm=l.split("'")[1]
        nm=nm[5:30]
        j=i+1
        while 'Used' not in L[j]: j+=1
        print(nm, L[i+2].strip()[:80] if 'spill' in L[i+2] else '', '|', L[j].split('Used')[1][:30])
