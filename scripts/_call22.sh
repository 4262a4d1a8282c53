python scripts/_dbg_p2p.py 2>&1 | head -40
