for st in 0 3000 6000 9000 12000; do echo "stagger $st"; STAGGER=$st MODE=nosync timeout 300 python tools/diag_step.py 2>&1 | tail -1; done
