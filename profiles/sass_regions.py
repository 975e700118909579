"""Static SASS instructions per function region of one kernel (leaf of the
inlined-at chain), from `nvdisasm --print-line-info-inline` output:

    nvcc ... -lineinfo -cubin -o k.cubin render.cu
    nvdisasm --print-line-info-inline k.cubin | awk '/^\\.text\\.<kernel>/{f=1} ...' > k.sass
    python profiles/sass_regions.py k.sass
"""
import collections
import re
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from inst_regions import region  # noqa: E402

leaf, fresh = None, True
cnt, tot = collections.Counter(), 0
for line in open(sys.argv[1]):
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        if fresh:
            leaf = (m.group(1).split("/")[-1], int(m.group(2)))
            fresh = False
        continue
    if re.match(r"^\s*/\*[0-9a-f]+\*/", line):
        tot += 1
        fresh = True
        if leaf:
            try:
                cnt[region(*leaf)] += 1
            except Exception:
                cnt[leaf[0]] += 1
print(tot, "SASS instructions")
for k, v in cnt.most_common(40):
    print(f"{v:6d} {k}")
