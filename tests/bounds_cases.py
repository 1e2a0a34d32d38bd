"""Out-of-bounds probe for the hot-path kernels (run by tests/test_gpu_bounds.py in a subprocess).

compute-sanitizer is not available on this GPU pool, so reads and writes past the end of the
caller's vectors are caught by the MMU instead: every vector handed to the C ABI is placed
with the CUDA virtual-memory API so that it ENDS at the end of its mapped range, with the next
2 MB of address space reserved but unmapped.  An access past the end is then an illegal-address
fault (sticky: hence the separate process).  16-byte alignment is required by the library, so
an odd-length vector ends 8 bytes before the boundary.  Results are compared bitwise with the
same calls on ordinary torch allocations.  HDGB_GRID_CAP=1 makes every CTA walk all element
groups and face batches.  Test infrastructure only.
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from cuda.bindings import driver as cu

    import paper_2007_11891_b200 as hb
    from paper_2007_11891_b200 import _lib
    from paper_2007_11891_b200.operator import DeviceContext

    torch.cuda.init()
    torch.zeros(1, device="cuda")
    L = _lib.lib()

    def ck(res):
        err = res[0] if isinstance(res, tuple) else res
        if err != cu.CUresult.CUDA_SUCCESS:
            raise RuntimeError(f"driver error {err}")
        return res[1] if isinstance(res, tuple) and len(res) > 1 else None

    prop = cu.CUmemAllocationProp()
    prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = 0
    gran = ck(cu.cuMemGetAllocationGranularity(prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM))
    keep = []

    def edge(nd):
        """Device pointer of nd doubles ending at (or 8 bytes before) an unmapped boundary."""
        nbytes = (8 * nd + 15) // 16 * 16
        size = (nbytes + gran - 1) // gran * gran
        va = ck(cu.cuMemAddressReserve(size + gran, 0, 0, 0))
        h = ck(cu.cuMemCreate(size, prop, 0))
        ck(cu.cuMemMap(va, size, 0, h, 0))
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = 0
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        ck(cu.cuMemSetAccess(va, size, [acc], 1))
        keep.append((va, h, size))
        return int(va) + size - nbytes

    def put(ptr, host):
        ck(cu.cuMemcpyHtoD(ptr, np.ascontiguousarray(host, dtype=np.float64), host.size * 8))

    def get(ptr, nd):
        out = np.empty(nd)
        ck(cu.cuMemcpyDtoH(out, ptr, nd * 8))
        return out

    S = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    degrees = [int(v) for v in sys.argv[1:]] or [1, 2, 3, 8, 12, 13, 14, 15, 16]
    for p in degrees:
        for n_el, bc in (((2, 1, 1), ("neumann", "dirichlet", "neumann", "neumann", "dirichlet", "neumann")),
                         ((3, 2, 2), ("dirichlet", "neumann", "neumann", "dirichlet", "dirichlet", "neumann")),
                         ((4, 3, 2), "dirichlet")):
            mesh = hb.Mesh(n_el, (0, 0, 0), (1.5, 1.0, 1.0), bc)
            dc = DeviceContext(hb.Basis1D(p, 0.7), mesh, 0.4)
            na, nu = dc.n_all, dc.n_unknown
            u = np.random.default_rng(p).uniform(-1, 1, na)
            pu, pr = edge(na), edge(na)
            put(pu, u)
            ut = torch.from_numpy(u).cuda()
            checks = 0
            for variant in (0, 1):
                _lib.check(L.hdgb_op_apply(dc.handle, variant, ctypes.c_void_p(pu), ctypes.c_void_p(pr), S))
                torch.cuda.synchronize()
                assert np.array_equal(get(pr, na), dc.apply(ut, variant).cpu().numpy()), ("apply", p, variant)
                checks += 1
            for kind in (1, 2, 3):
                _lib.check(L.hdgb_prec_apply(dc.handle, kind, ctypes.c_void_p(pu), ctypes.c_void_p(pr), S))
                torch.cuda.synchronize()
                assert np.array_equal(get(pr, na), dc.prec(ut, kind).cpu().numpy()), ("prec", p, kind)
                checks += 1
            A = np.ascontiguousarray(dc_T := np.random.default_rng(1).standard_normal((p + 1, p + 1)))
            _lib.check(L.hdgb_face_transform(dc.handle, ctypes.c_void_p(A.ctypes.data), ctypes.c_void_p(pu),
                                             ctypes.c_void_p(pr), S))
            torch.cuda.synchronize()
            assert np.array_equal(get(pr, na), dc.transform(ut, dc_T).cpu().numpy()), ("transform", p)
            pk = edge(nu)
            _lib.check(L.hdgb_pack(dc.handle, ctypes.c_void_p(pu), ctypes.c_void_p(pk), S))
            _lib.check(L.hdgb_unpack(dc.handle, ctypes.c_void_p(pk), ctypes.c_void_p(pr), S))
            torch.cuda.synchronize()
            F = get(pr, na)
            assert np.array_equal(F, dc.unpack(dc.pack(ut)).cpu().numpy()), ("pack", p)
            for variant, kind in ((0, 1), (1, 3), (0, 0)):
                px = edge(na)
                put(px, np.zeros(na))
                it, rel, conv = ctypes.c_int32(), ctypes.c_double(), ctypes.c_int32()
                _lib.check(L.hdgb_pcg(dc.handle, variant, kind, ctypes.c_void_p(pr), ctypes.c_void_p(px), 1e-10, 0.0,
                                      200, ctypes.byref(it), ctypes.byref(rel), ctypes.byref(conv), S))
                torch.cuda.synchronize()
                xt = torch.zeros(na, dtype=torch.float64, device="cuda")
                it2, _, _ = dc.pcg(variant, kind, torch.from_numpy(F).cuda(), xt, 1e-10, 0.0, 200)
                assert it.value == it2 and np.array_equal(get(px, na), xt.cpu().numpy()), ("pcg", p, variant, kind)
                checks += 1
            print(f"p={p} n_el={n_el} n_all={na} ({'odd' if na % 2 else 'even'}) {checks} checks ok", flush=True)
            del dc
    print("OK")


if __name__ == "__main__":
    main()
