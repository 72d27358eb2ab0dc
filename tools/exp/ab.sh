for r in 1 2 3; do
python tools/exp_ab.py time 16384 16384 16384 base nofk old
python tools/exp_ab.py time 16384 16384 4096 base nofk old
python tools/exp_ab.py time 4096 4096 4096 base nofk old
done
