timeout 600 python profiles/kexp.py time tpriv --cfg c2 --reps 5
