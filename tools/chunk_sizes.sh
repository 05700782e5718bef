# kernel and step time of one cfg3 field call at the e2e chunk sizes (fractions of a 9,472-candidate wave)
for b in 1184 2368 4736 7104 8704 9472 18944; do
  timeout 120 python bench.py --batch $b --no-extras --steps 30 > gpurun_out/chunk_$b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/chunk_$b.json').read().strip().splitlines()[-1])
print($b, round($b/9472,3), 'step', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4), 'launches', d.get('gpu_launches'))"
done
