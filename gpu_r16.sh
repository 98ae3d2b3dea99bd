./profiles/mb_tma
