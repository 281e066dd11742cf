for cfg in "0 0" "16 0" "11 0" "0 32" "16 32" "8 21"; do set -- $cfg
  echo "== PRE_ZC=$1 POST_ZC=$2"
  PINT_3D_PRE_ZC=$1 PINT_3D_POST_ZC=$2 timeout 300 python tools/bench_cfg.py --config c3 --steps 5 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
k = d['kernels']
print('ms/iter %.3f  post_fine %.3f  pre_fine %.3f  post_coarse %.3f  pre_coarse %.3f' % (d['ms_per_iter'], k['mg_post_fine']['ms'], k['mg_pre_fine']['ms'], k['mg_post_coarse']['ms'], k['mg_pre_coarse']['ms']))"
done
