import ctypes as C
lib = C.CDLL('./debug/libmmabench.so')
out = (C.c_longlong * 2)()
print("N mode nblk issue total cyc/mma ideal")
for N, modes in ((32, (11,)), (96, (11,)), (256, (11,))):
    for mode in modes:
        for nb in (1, 148):
            rows = 400
            rc = lib.run_mma_bench(N, mode, rows, nb, out)
            print(N, mode, nb, out[0], out[1], round(out[1] / (rows * 6), 1), N * 128 // 256, "rc", rc)
