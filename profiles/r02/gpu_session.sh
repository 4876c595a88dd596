PT_T=131072 PT_DECODE=1 python profiles/phase_timers.py
PT_T=131072 PT_DECODE=16 python profiles/phase_timers.py
