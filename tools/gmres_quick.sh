#!/bin/bash
# quick GMRES timing set: cfg1, cfg4 (c128/c64) and the cfg2 bench solve times
timeout 600 python tools/bench_configs.py cfg4 cfg1 > /dev/null 2>&1
python -c "import json; d=json.load(open('gpurun_out/configs.json')); print('cfg1', d['cfg1']['gmres']['none']['ms'], d['cfg1']['gmres']['pk']['ms'], 'cfg4', d['cfg4_complex128']['gmres']['none']['ms'], d['cfg4_complex128']['gmres']['pk']['ms'], d['cfg4_complex64']['gmres']['none']['ms'], d['cfg4_complex64']['gmres']['pk']['ms'])"
python bench.py --steps 300 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', d['value'], [(k,v['solve_ms']) for k,v in d['config']['gmres'].items()])"
