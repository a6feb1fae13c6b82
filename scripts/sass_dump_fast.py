"""Print the fast path of one kernel's main walk loop (see sass_fastpath.py)."""
import re
import sys

text = open(sys.argv[1]).read()
for part in re.split(r'\n\s*Function : ', text)[1:]:
    name = part.split('\n', 1)[0].strip()
    if sys.argv[2] not in name:
        continue
    L = [re.sub(r'\s*/\* 0x[0-9a-f]+ \*/\s*$', '', l.strip()) for l in part.split('\n')
         if re.match(r'\s*/\*[0-9a-f]{4,5}\*/', l)]
    A = [int(re.match(r'/\*([0-9a-f]+)\*/', l).group(1), 16) for l in L]
    pos = {a: i for i, a in enumerate(A)}
    loops = []
    for i, l in enumerate(L):
        m = re.search(r'BRA (0x[0-9a-f]+)', l)
        if m:
            t = int(m.group(1), 16)
            if t < A[i]:
                loops.append((t, A[i], i))
    # argv[3]: which loop, by size rank (0 = the largest)
    loops.sort(key=lambda x: x[0] - x[1])
    t0, t1, iend = loops[int(sys.argv[3]) if len(sys.argv) > 3 else 0]
    i = pos[t0]
    while i <= iend:
        l = L[i]
        print(l.split('*/', 1)[1].strip()[:80])
        m = re.search(r'@!?P\d BRA (!?P\d, )?(0x[0-9a-f]+)', l)
        if m:
            t = int(m.group(2), 16)
            if t > A[i] and any('0x3d719799' in x or '0x812dea11' in x for x in L[i + 1:i + 6]):
                print('   ... slow path ...')
                i = pos[t]
                continue
        i += 1
    break
