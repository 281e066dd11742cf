# A/B of 3D band-kernel occupancy variants (libpint_<V>.so built with -DPINT_C3T/... macros)
for v in "" _B _C _D _F; do
  echo "== variant ${v:-A}"
  PINT_LIB=$PWD/paper_1802_08126_b200/libpint$v.so timeout 300 python tools/bench_cfg.py --config c3 --steps 5 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
k = d['kernels']
print('ms/iter %.3f  post_fine %.3f  pre_fine %.3f  post_coarse %.3f  pre_coarse %.3f' % (d['ms_per_iter'], k['mg_post_fine']['ms'], k['mg_pre_fine']['ms'], k['mg_post_coarse']['ms'], k['mg_pre_coarse']['ms']))"
done
