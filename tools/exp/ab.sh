for r in 1 2 3; do
python tools/exp_ab.py time 4096 4096 4096 base pf4 pf8 pf16
python tools/exp_ab.py time 16384 16384 4096 base pf4 pf8 pf16
python tools/exp_ab.py time 16384 16384 16384 base pf8
done
