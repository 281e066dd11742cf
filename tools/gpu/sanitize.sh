# compute-sanitizer racecheck / synccheck / memcheck over the band-kernel tests
# (2D cells 128 / 256, 3D cells 16 / 32): the kernels hand-manage mbarrier
# rings, halo rows and zero-padded slices.
set -x
SEL2D="tests/test_gpu_parity.py::test_band_levels_bitwise tests/test_gpu_parity.py::test_band_uzawa_matches_oracle"
SEL3D="tests/test_gpu_3d.py::test_operators_and_preconditioners_3d"
for tool in racecheck synccheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest $SEL2D -x -q -k "not 512" > gpurun_out/sanitizer_${tool}_2d.log 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_${tool}_2d.log
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest $SEL3D -x -q -k "16 or 32" > gpurun_out/sanitizer_${tool}_3d.log 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_${tool}_3d.log
done
tail -4 gpurun_out/sanitizer_*.log
