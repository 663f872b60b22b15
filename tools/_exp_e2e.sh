# e2e host-pipeline chunk counts (DIS_HOST_CHUNKS)
cd $GRAFT_REPO_ROOT
for n in ${CHUNKS:-4 8 12 16}; do
  DIS_HOST_CHUNKS=$n timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 10 --config ${CFG:-c1} 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('chunks $n value %.0f e2e %.0f e2e_ms %.2f' % (d['value'], d['e2e']['value'], d['e2e']['ms_per_step']))"
done
