# DST data-path A/B on c2: PINT_DST_DEBUG bit 0 = movement only, bit 2 = 8-byte path
for dbg in 0 4 1 5; do
PINT_DST_DEBUG=$dbg timeout 600 python tools/kstats_c2.py 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print('PINT_DST_DEBUG=%s step %.3f  S^T %.4f  S %.4f' % (d['env'].get('PINT_DST_DEBUG'), d['ms_per_step'], d['ms']['dst_inverse_transpose'], d['ms']['dst_inverse']))"
done
