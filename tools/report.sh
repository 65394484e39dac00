#!/bin/bash
# summarise an iteration: tests, bench line, leaf-kernel ncu summary and hot lines
cd /root/repo
tail -2 gpurun_out/it_pytest.log
python3 -c "
import json,sys
for l in open('gpurun_out/it_bench.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('value %.3g samples/s  ms/step %.2f  leaf %.2f ms  split %.2f ms  frac %.3f  clocks %s' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['split_ms'], r['frac'], d['clocks']))
"
tail -1 gpurun_out/it_bench.log | grep -v '^{'
ncu -i gpurun_out/it_prof.ncu-rep --page details --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
mi=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
want=['Duration','Registers Per Thread','Achieved Occupancy','Executed Ipc Active','Issue Slots Busy','Executed Instructions','DRAM Throughput']
print('  '.join(f'{x[mi]}={x[vi]}{x[ui]}' for x in r[1:] if x[mi] in want))
"
ncu -i gpurun_out/it_prof.ncu-rep --page source --csv --kernel-name regex:k_leaf --print-source cuda,sass > /tmp/it_src.csv 2>&1
python3 tools_ncu_lines.py /tmp/it_src.csv ${1:-20}
