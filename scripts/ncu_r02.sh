set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r02_launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r02_ncu_launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_sell_op|k_to_internal|k_fill" -s 6 -c 3 -o gpurun_out/r02_c2 python scripts/xperm_probe.py 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pcg_matvec -s 6 -c 1 -o gpurun_out/r02_c3p python scripts/c3p_ncu_target.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_jacobi_step -s 6 -c 1 -o gpurun_out/r02_c4 python scripts/jacobi_ncu_target.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pcg_matvec|k_pcg_update|k_pcg_direction" -s 12 -c 3 -o gpurun_out/r02_c5 python scripts/pcg_ncu_target.py 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_vec_cg1_update|k_dist_matvec_sweep|k_dist_q_iface" -s 8 -c 3 -o gpurun_out/r02_dist_c5 python scripts/dist_ncu_target.py 5 > /dev/null 2>&1
ls -la gpurun_out/
