import ctypes as C, os, sys
lib = C.CDLL(os.path.join(os.environ.get("GRAFT_REPO_ROOT","/root/repo"), "paper_2604_17861_b200/lib/libgpuos_bench.so"))
lib.gb_config3.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
out = (C.c_double * 16)()
for dt in (0, 4):
    lib.gb_config3(0, dt, 20, out)
    print(os.environ.get("GB_WORKERS"), dt, "step", round(out[0],1), "phases", [round(out[5+i],1) for i in range(4)])
