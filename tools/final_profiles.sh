# Final-build evidence of a round: GPU suite, bench line, launch list + traffic of one bench
# step, full ncu report of the Jacobi kernel, secondary-kernel rooflines, config times.
# Usage (on the GPU box): bash tools/final_profiles.sh <tag>   -> gpurun_out/<tag>_*
set -x
cd $GRAFT_REPO_ROOT
T=${1:-r02f}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; tail -2 gpurun_out/${T}_pytest.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -c 600 gpurun_out/${T}_bench.json
python tools/profile_step.py --replicas 8 > gpurun_out/${T}_step_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__ops_path_tensor_src_fp64.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${T}_step_launches.csv python tools/profile_step.py --replicas 8 > gpurun_out/${T}_step_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/${T}_step_launches.csv | head -20
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:jacobi_dynamic -c 1 -o gpurun_out/${T}_jacobi_full -f python tools/profile_step.py --replicas 8 > gpurun_out/${T}_full_ncu.log 2>&1; tail -2 gpurun_out/${T}_full_ncu.log
python tools/kernel_rooflines.py --launch-list gpurun_out/${T}_step_launches.csv > gpurun_out/${T}_kernel_rooflines.json 2> gpurun_out/${T}_kr.err; tail -c 800 gpurun_out/${T}_kernel_rooflines.json
python tools/config_times.py > gpurun_out/${T}_configs.log 2>&1; tail -3 gpurun_out/${T}_configs.log
