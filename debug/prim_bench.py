import ctypes as C
lib = C.CDLL('./debug/libprim.so')
out = (C.c_longlong * 6)()
for busy in (0, 1):
    rc = lib.run_prim(2000, busy, out)
    print("busy", busy, "rc", rc, dict(zip(["ld16+wait", "st16+wait+fence", "2xSTS", "fence.proxy.async", "syncwarp+arrive", "trywait(done)+syncwarp"], list(out))))
