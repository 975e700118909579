"""Static SASS size per source line of one kernel (nvdisasm -gi line info).

usage: python profiles/sass_lines.py FILE.cubin KERNEL_SUBSTR [outer_file] [topN]
Counts instructions per leaf (file, line) and per outermost frame in
`outer_file` (inlined-at chain), to find what bloats the instruction cache.
"""
import collections, re, subprocess, sys

cubin, kname = sys.argv[1], sys.argv[2]
outer_file = sys.argv[3] if len(sys.argv) > 3 else None
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
txt = subprocess.run(["nvdisasm", "--print-line-info-inline", cubin],
                     capture_output=True, text=True).stdout
leaf, outer, fn = None, None, None
lc, oc, tot = collections.Counter(), collections.Counter(), 0
for l in txt.splitlines():
    if l.startswith(".text."):
        fn = l
    if "//## File" in l:
        frames = [(f.split("/")[-1], int(n))
                  for f, n in re.findall(r'File "([^"]+)", line (\d+)', l)]
        leaf = frames[0]
        ob = [fr for fr in frames if outer_file and fr[0] == outer_file]
        outer = ob[-1] if ob else leaf
        continue
    if fn and kname in fn and re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+[A-Z@]", l):
        lc[leaf] += 1
        oc[outer] += 1
        tot += 1
print(f"{kname}: {tot} SASS instructions")
print("-- by leaf line")
for k, c in lc.most_common(top):
    print(f"{c:6d} {k[0]}:{k[1]}")
if outer_file:
    print(f"-- by outermost {outer_file} frame")
    for k, c in oc.most_common(top):
        print(f"{c:6d} {k[0]}:{k[1]}")
