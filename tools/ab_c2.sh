mkdir -p gpurun_out
for cfg in "GN_LIB=exp/libgnb200_s0.so GN_SMEM_RES_KB=0" "GN_LIB=exp/libgnb200_na.so GN_SMEM_RES_KB=0" "GN_LIB=exp/libgnb200_s0.so GN_SMEM_RES_KB=0 GN_PLAN_COLOCATE=1" "GN_LIB=exp/libgnb200_na.so GN_SMEM_RES_KB=0 GN_PLAN_COLOCATE=1"; do
  echo "== $cfg"
  env $cfg python tools/probe.py --which C2,C3 --grid 0 --iters 1000 --reps 2 --dtypes fp64 2>&1 | grep -v "^#"
done
M=gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum
env GN_LIB=exp/libgnb200_na.so GN_SMEM_RES_KB=0 GN_PLAN_COLOCATE=1 ncu --metrics $M --clock-control none -k regex:k_gn_loop -c 1 --csv python tools/probe.py --which C2 --grid 0 --iters 100 --reps 1 --dtypes fp64 2>&1 | grep '"14"\|"1[0-9]",' | cut -d, -f12-
