for lib in paper_2405_17381_b200/libla_b200.so build/var/libmc2.so build/var/libmc1.so; do
echo "$lib"; LA_B200_LIB=$lib TL_H=4 TL_D=64 TL_DTYPE=f32 timeout 200 python tools/timeline.py 1:1024 2>&1 | grep "=="
done
