EXP_ACC=1 EXP_REPS=3 python tools/exp_ab.py time 4096 4096 4096 base stg2
EXP_ACC=1 EXP_REPS=3 python tools/exp_ab.py time 4000 4040 1000 base stg2
for r in 1 2 3; do
python tools/exp_ab.py time 4096 4096 4096 base stg2 nostore
python tools/exp_ab.py time 16384 16384 4096 base stg2 nostore
done
python tools/exp_ab.py time 4096 4096 4096 stg2tr
