for r in 1 2; do
for ag in 1 0; do echo -n "cfg4 ag=$ag: "; CTF_FSPLIT_AG=$ag timeout 300 python tools/prof_cfg.py --cfg 4 --iters 2 2>&1 | tail -1; done
for ag in 1 0; do echo -n "cfg3 ag=$ag: "; CTF_FSPLIT_AG=$ag timeout 300 python tools/prof_cfg.py --cfg 3 --iters 2 2>&1 | tail -1; done
done
for c in 3 4; do CTF_DEV_LIB=tools/dev/fph/libctfiss.so timeout 300 python tools/fsplit_phase.py --cfg $c 2>&1 | tail -10; done
