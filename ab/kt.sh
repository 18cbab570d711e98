#!/bin/bash
# per-kernel durations (ncu) of one fill: ab/kt.sh ENGINE DIST LOG2N [params]
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/profile_fill.py "$@" --reps 2 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
d={}
for r in rows[1:]:
    d.setdefault(r[ki].split('(')[0][-28:],{})[r[mi].split('__')[1][:14]]=r[vi]
for k,v in d.items(): print('%-30s'%k, v)
"
