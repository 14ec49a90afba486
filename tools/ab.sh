for v in old new old new; do
RT3D_LIB=$PWD/ab_$v.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_classes']
print('$v', round(d['value'],1), round(d['e2e']['value'],1), 'apss', round(k['apss']['us_per_launch'],1), 'knn', round(k['knn']['us_per_launch'],1), 'tail', round(k['stage_tail']['us_per_launch'],1))"
done
