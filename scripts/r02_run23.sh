#!/bin/bash
# full GPU suite + smoke + default bench on the current build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke23.txt 2>&1
tail -1 gpurun_out/smoke23.txt
timeout 3600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_r23.txt 2>&1
tail -3 gpurun_out/pytest_r23.txt
timeout 900 python bench.py > gpurun_out/bench23.json 2> gpurun_out/bench23.err
python -c "import json;d=json.load(open('gpurun_out/bench23.json'));print(d['value'], d['undivided_ms_per_step'], d['speedup_vs_undivided'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['plan_seconds'], d['steps'])"
timeout 900 python bench.py --net resnet18 --no-cpu --steps 20 > gpurun_out/r18_23.json 2> gpurun_out/r18_23.err
timeout 900 python bench.py --net resnet50 --mode wd --total-mib 2544 --no-cpu --steps 10 > gpurun_out/r50_23.json 2> gpurun_out/r50_23.err
for f in r18_23 r50_23; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['value'], d['undivided_ms_per_step'], d['speedup_vs_undivided'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"; done
