# sustained-load A/B (power cap regime): 40 steps each, alternating
for rep in 1 2; do for v in base sleep; do
lib=paper_2405_17381_b200/libla_b200.so; [ $v = sleep ] && lib=build/var/libsleep.so
LA_B200_LIB=$lib timeout 300 python tools/step_probe.py 40 > gpurun_out/sp_${v}_$rep.log 2>&1
done; done
