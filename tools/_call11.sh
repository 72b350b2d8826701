timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_cabi.py tests/test_gpu_faults.py -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/gputest11.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest11.log
for z in 1 0 1 0; do
CF_TAB_ZC=$z timeout 300 python bench.py --config C1 --steps 100 --skip-extras --skip-schemes --skip-cpu-baseline --skip-chase > gpurun_out/bench11_C1_z$z.json 2>gpurun_out/bench11_C1_z$z.err
python -c "
import json; d=json.loads(open('gpurun_out/bench11_C1_z$z.json').read().strip().splitlines()[-1]); e=d['e2e']; print('zc=$z', e['ms_per_step'], e['frac_of_link_roofline'], e['host_link_same_size_gbs'])"
done
