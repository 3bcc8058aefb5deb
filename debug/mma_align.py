import ctypes as C
lib = C.CDLL('./debug/libmmaalign.so')
out = (C.c_longlong * 2)()
for mode in (0, 1, 2, 3):
    for shift in (1,):
        for nb in (148,):
            n = 200
            rc = lib.run(shift, n, nb, out, mode)
            print(f"mode {mode} (0 back-to-back, 1 commit per batch, 2 two in flight, 3 one in flight) shift {shift} blocks {nb}: {out[0] / (n * 18):.1f} cycles per MMA  rc {rc}")
