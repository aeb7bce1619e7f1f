set -x
cd $GRAFT_REPO_ROOT
# 1. compute-sanitizer probe (one tool, smallest case, bounded)
( timeout 300 compute-sanitizer --tool memcheck python tools/sanitize_case.py --part queries > gpurun_out/r02_sanitizer_probe.log 2>&1; echo "exit $?" >> gpurun_out/r02_sanitizer_probe.log ) 
tail -5 gpurun_out/r02_sanitizer_probe.log
# 2. invariant-check build over the whole GPU suite, the bench and the stress loop
BMPS_LIB=tools/variants/debugchecks.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_debugchecks_pytest.log 2>&1; tail -2 gpurun_out/r02_debugchecks_pytest.log
BMPS_LIB=tools/variants/debugchecks.so timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/r02_debugchecks_bench.json 2> gpurun_out/r02_debugchecks_bench.err; grep -c BMPS_CHECK gpurun_out/r02_debugchecks_bench.err
BMPS_LIB=tools/variants/debugchecks.so timeout 600 python tools/debug_stress.py 25 > gpurun_out/r02_debugchecks_stress.log 2>&1; tail -2 gpurun_out/r02_debugchecks_stress.log
# 3. launch list with traffic metrics of one bench step (8 replicas)
python tools/profile_step.py --replicas 8 > gpurun_out/s4_step_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__ops_path_tensor_src_fp64.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02_step_launches.csv python tools/profile_step.py --replicas 8 > gpurun_out/s4_step_ncu.log 2>&1
tail -2 gpurun_out/s4_step_plain.log; tail -2 gpurun_out/s4_step_ncu.log
python tools/launch_summary.py gpurun_out/r02_step_launches.csv | head -20
# 4. full-set capture of the Jacobi kernel (one launch)
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:jacobi_dynamic -c 1 -o gpurun_out/r02_jacobi_full -f python tools/profile_step.py --replicas 8 > gpurun_out/s4_full_ncu.log 2>&1; tail -2 gpurun_out/s4_full_ncu.log
ls -la gpurun_out/*.ncu-rep
# 5. secondary kernels' rooflines and all configs end to end
python tools/kernel_rooflines.py --launch-list gpurun_out/r02_step_launches.csv > gpurun_out/r02_kernel_rooflines.json 2> gpurun_out/s4_kr.err; tail -c 1500 gpurun_out/r02_kernel_rooflines.json
python tools/config_times.py > gpurun_out/r02_configs.log 2>&1; tail -6 gpurun_out/r02_configs.log
