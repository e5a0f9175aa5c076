#!/bin/bash
# Source lines of the local-memory spills (STL/LDL) of one kernel: tools/spills.sh <regex of kernel>
set -e
D=$(mktemp -d)
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -I/root/repo/include \
  -I/root/repo/paper_1603_08390_b200/csrc --expt-relaxed-constexpr -cubin \
  /root/repo/paper_1603_08390_b200/csrc/genie_query.cu -o $D/q.cubin
nvdisasm --print-line-info $D/q.cubin > $D/q.sass
python3 - "$D/q.sass" "$1" <<'PY'
import re, sys
fn = None; line = None; res = {}
for l in open(sys.argv[1]):
    m = re.match(r'\s*\.text\.(\S+):', l)
    if m: fn = m.group(1)
    m = re.search(r'line (\d+)', l)
    if m and '//##' in l: line = (l.split('"')[1].rsplit('/', 1)[-1] if '"' in l else '?') + ':' + m.group(1)
    if fn and re.search(sys.argv[2], fn) and re.search(r'\b(STL|LDL)', l):
        k = ('STL' if 'STL' in l else 'LDL', line); res[k] = res.get(k, 0) + 1
for k, v in sorted(res.items(), key=lambda x: -x[1]): print(v, *k)
PY
rm -rf $D
