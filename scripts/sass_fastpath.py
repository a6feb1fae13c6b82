"""Fast-path instruction count of each kernel's main walk loop (the largest
backward branch), skipping the exact-voxel slow path, from cuobjdump -sass."""
import collections
import re
import sys

text = open(sys.argv[1]).read()
for part in re.split(r'\n\s*Function : ', text)[1:]:
    name = part.split('\n', 1)[0].strip()
    L = [re.sub(r'\s*/\* 0x[0-9a-f]+ \*/\s*$', '', l.strip()) for l in part.split('\n')
         if re.match(r'\s*/\*[0-9a-f]{4,5}\*/', l)]
    A = [int(re.match(r'/\*([0-9a-f]+)\*/', l).group(1), 16) for l in L]
    pos = {a: i for i, a in enumerate(A)}
    loops = []
    for i, l in enumerate(L):
        m = re.search(r'BRA (0x[0-9a-f]+)', l)
        if m:
            t = int(m.group(1), 16)
            if t < A[i] and (A[i] - t) // 16 > 150:
                loops.append((t, A[i], i))
    for t0, t1, iend in loops:
        if t0 not in pos:
            continue
        i, seq = pos[t0], []
        while i <= iend:
            l = L[i]
            seq.append(l)
            m = re.search(r'@!?P\d BRA (!?P\d, )?(0x[0-9a-f]+)', l)
            if m:
                t = int(m.group(2), 16)
                if t > A[i] and any('0x3d719799' in x or '0x812dea11' in x for x in L[i + 1:i + 6]):
                    i = pos[t]
                    continue
            i += 1
        if not any('LDG' in x for x in seq):
            continue  # a setup loop, not a walk
        c = collections.Counter(re.sub(r'^@!?P\d\s+', '', x.split('*/', 1)[1].strip()).split(' ')[0].split('.')[0]
                                for x in seq)
        print(name[:40], 'loop', (t1 - t0) // 16 + 1, 'fast', len(seq), sorted(c.items(), key=lambda x: -x[1]))
