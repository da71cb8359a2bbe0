echo "rel1 $(LA_B200_LIB=build/var/librel1.so timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)"
for rep in 1 2 3; do for lib in paper_2405_17381_b200/libla_b200.so build/var/librel1.so; do echo "$lib $(LA_B200_LIB=$lib timeout 120 python tools/exp_time.py 2>&1 | tail -1)"; done; done
