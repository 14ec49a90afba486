for k in B C; do echo "== $k"; RT3D_LIB=$PWD/ab_prof.so timeout 300 python tools/sweep_profile.py $k 2>&1 | head -30; done
