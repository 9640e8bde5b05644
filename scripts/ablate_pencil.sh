set -x
for f in "" "-DVIE_ABL_NOHAD" "-DVIE_ABL_NOFFT" "-DVIE_ABL_NOHAD -DVIE_ABL_NOFFT"; do
  python -c "
import sys; sys.path.insert(0,'.')
from paper_1811_00484_b200 import build
build.build(force=True, extra='$f'.split())
" && python bench.py --config head_2mm --steps 5 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['stage_ms']['pencil'])"
done
