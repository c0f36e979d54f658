for n in 1600000 3200000 6300000 12700000 25000000; do python tools/time_kernels.py --n $n --reps 10 | cut -c1-200; done
