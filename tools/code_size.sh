#!/bin/bash
# code size per function of the product kernel
cd /root/repo/paper_2603_17456_b200/csrc
cuobjdump -xelf all /root/repo/build/obj/device/engine_kernel.o -o /tmp >/dev/null 2>&1
cd /tmp && cuobjdump -xelf all /root/repo/build/obj/device/engine_kernel.o >/dev/null 2>&1
nvdisasm -c /tmp/engine_kernel.sm_100a.cubin > /tmp/ek.sass 2>&1
python3 - <<'PY'
import re, subprocess
lines=open('/tmp/ek.sass').read().split('\n')
cur='kernel'; cnt={}
for l in lines:
    m=re.match(r'^\$_ZN3mfb19mfsim_engine_kernel[^$]*\$(\S+):',l)
    if m: cur=m.group(1); continue
    if re.match(r'^\s+/\*[0-9a-f]{4,}\*/',l): cnt[cur]=cnt.get(cur,0)+1
tot=sum(cnt.values())
for k,v in sorted(cnt.items(), key=lambda kv:-kv[1])[:int(__import__('os').environ.get('TOP','30'))]:
    dn=subprocess.run(['c++filt',k],capture_output=True,text=True).stdout.strip()
    dn=re.sub(r'mfb::Engine<mfb::WarpLanes, false, (true|false)>::',lambda m:('C:' if m.group(1)=='true' else 'G:'),dn)
    print(f'{v*16/1024:7.1f}KB  {dn[:100]}')
print(f'total {tot*16/1024:.0f} KB')
PY
