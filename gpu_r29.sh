for bs in 16 32 64; do timeout 120 python profiles/time_step.py 32 52 52 8192 128 $bs; done
for bs in 16 64; do timeout 120 python profiles/time_step.py 32 52 52 512 128 $bs; done
