#!/bin/bash
# usage: spills.sh [extra nvcc flags]; prints spill summary + top local-memory lines of ed_persistent_bf16
cd /root/repo/paper_2302_03851_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include -I. "$@" -Xptxas -v -cubin -o /tmp/k.cubin ed_kernels.cu 2>&1 | grep -A2 "properties for _ZN2ed18ed_persistent_bf16" | tail -2
nvdisasm -g /tmp/k.cubin > /tmp/all_li.sass 2>&1
python3 - <<'PY'
import re, collections
cur=None; c=collections.Counter(); infn=False
src=open('/root/repo/paper_2302_03851_b200/csrc/ed_kernels.cu').read().splitlines()
for l in open('/tmp/all_li.sass'):
    if '.text._ZN2ed18ed_persistent_bf16' in l and ':' in l: infn=True
    elif '.text.' in l and ':' in l and 'bf16ENS' not in l: infn=False
    m=re.search(r'line (\d+)',l)
    if m: cur=int(m.group(1))
    if infn and re.search(r'\b(STL|LDL)\b',l): c[cur]+=1
tot=sum(c.values())
print("local ops", tot)
for k,v in sorted(c.items(), key=lambda kv:-kv[1])[:14]: print(f"{v:5d} {k}: {src[k-1].strip()[:110]}")
PY
