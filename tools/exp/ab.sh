for r in 1 2 3; do
python tools/exp_ab.py time 16384 16384 16384 base mma1
python tools/exp_ab.py time 16384 16384 4096 base mma1
python tools/exp_ab.py time 4096 4096 4096 base mma1
done
EXP_ACC=1 EXP_REPS=3 python tools/exp_ab.py time 4096 4096 4096 base mma1
