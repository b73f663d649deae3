#!/bin/bash
# build an A/B variant of the library: tools/ab_build.sh NAME [extra nvcc flags...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
python - "$name" "$@" <<'PY'
import subprocess, sys, pathlib
sys.path.insert(0, '.')
import __graft_entry__ as g
name, extra = sys.argv[1], sys.argv[2:]
srcs = sorted(pathlib.Path('paper_2605_06374_b200/csrc').glob('*.cu'))
out = pathlib.Path('tools/ab') / f'lib_{name}.so'
procs = []
objs = []
for s in srcs:
    o = pathlib.Path('tools/ab') / f'{name}_{s.stem}.o'
    objs.append(str(o))
    procs.append(subprocess.Popen(['/usr/local/cuda/bin/nvcc', *g.NVCC_FLAGS, *extra, '-c', str(s), '-o', str(o)]))
assert all(p.wait() == 0 for p in procs)
subprocess.check_call(['/usr/local/cuda/bin/nvcc', '-gencode', 'arch=compute_100a,code=sm_100a', '-shared', *objs, '-o', str(out)])
for o in objs: pathlib.Path(o).unlink()
print(out)
PY
