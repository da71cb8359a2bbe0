for v in rel1 rel2; do echo "$v $(LA_B200_LIB=build/var/lib$v.so timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)"; done
bash tests/gpu_ab_bench.sh 2 paper_2405_17381_b200/libla_b200.so build/var/librel1.so build/var/librel2.so
