# e2e leg with edge pieces: correctness test + a default bench run
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r3p; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_execute.py -q -x -k "e2e or graph" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 600 $O/bench.err
python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], json.dumps(d['e2e'])[:300], d['clocks'])"
