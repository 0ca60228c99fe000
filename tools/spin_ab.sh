# Spin vs sleep waits (LUTGPU_OH_SPIN) and the watcher (LUTGPU_OH_WATCH) under sustained load (40 steps: the power cap
# engages), with the SM clock histogram.  Needs a probe variant of onehot.cu: tools/build_variant.sh onehot.cu p -DLUTGPU_PROBES
cd /root/repo
for s in 3 0 3 0; do
  LUTGPU_OH_SPIN=$s LUTGPU_LIB=paper_2302_03213_b200/_lib/liblutgpu_p.so timeout 200 python bench.py --no-cpu --no-variants --no-ties --no-e2e --steps 40 --warmup 3 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);c=d['clocks'];print('spin=$s', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['roofline']['kernel_ms'].items()}, c['sm_mhz_hist'], c['reasons'], c['power_w_max'])"
done
for w in 1 0; do
  LUTGPU_OH_WATCH=$w LUTGPU_LIB=paper_2302_03213_b200/_lib/liblutgpu_p.so timeout 200 python bench.py --no-cpu --no-variants --no-ties --no-e2e --steps 40 --warmup 3 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);c=d['clocks'];print('watch=$w', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['roofline']['kernel_ms'].items()}, c['sm_mhz_hist'], c['reasons'])"
done
