"""Thin Python binding of the C-ABI in include/pf.h (argument marshalling only).

Every step of the hot path runs in libpf.so's sm_100a kernels; this module
only checks tensor dtypes/devices, passes raw pointers and the current CUDA
stream, and raises on a non-PF_OK status.  There is no CPU fallback: if the
extension is missing or no CUDA device is visible, calls fail loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("PF_LIB") or os.path.join(_HERE, "libpf.so")  # PF_LIB: experiment builds

PF_OK, PF_ERR_ARG, PF_ERR_TOPOLOGY, PF_ERR_CAPACITY, PF_ERR_CUDA, PF_ERR_STATE = range(6)
_STATUS = {1: "PF_ERR_ARG", 2: "PF_ERR_TOPOLOGY", 3: "PF_ERR_CAPACITY", 4: "PF_ERR_CUDA", 5: "PF_ERR_STATE"}

STRUCTURE = dict(x_theta=0, x_v=1, u_v=2, u_p=3, gx_ptr=4, gx_idx=5, gu_ptr=6, gu_idx=7, a_ptr=8, a_idx=9,
                 bus_order=10, perm=11, block_ptr=12, lu_ptr=13, lu_idx=14, level_l_ptr=15, level_l_blk=16,
                 level_u_ptr=17, level_u_blk=18, front_row=19, lu_subtree_ptr=20, lu_subtree_blk=21,
                 lu_level_blk=22)

# exported symbols declared in include/pf.h
SYMBOLS = ["pf_build_network", "pf_build_network_ex", "pf_destroy", "pf_query", "pf_get_structure", "pf_last_error", "pf_build_error",
           "pf_eval_constraints", "pf_jacobian", "pf_reduced_hessian_batch", "pf_condensed_kkt_solve",
           "pf_launch_count", "pf_profile", "pf_kernel_times", "pf_condensed_rhs", "pf_recover_step",
           "pf_power_flow", "pf_reduced_gradient", "pf_condensed_kkt_solve_reg"]


class PFError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (_STATUS.get(status, status), msg))
        self.status = status


class pf_dims(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "n_b", "n_l", "n_g", "n_x", "n_u", "m", "n_r", "n_h", "ref_bus", "ref_gen", "nnz_gx", "nnz_gu", "nnz_a",
        "nnz_lu", "n_blocks", "n_levels_l", "n_levels_u", "max_batch", "max_scen", "tile_cols",
        "reach_rows_l", "reach_rows_ua", "gu_rows", "front_level", "front_rows", "lu_cut_level", "lu_pairs")]


_lib = None


def load_library():
    """Load libpf.so (ctypes).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError("libpf.so not built: run `python -m paper_2203_11875_b200._build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(_LIB_PATH)
    P, I32, D, VP = ctypes.c_void_p, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p
    lib.pf_build_network.argtypes = [I32, I32, I32] + [P] * 8 + [I32] + [P] * 5 + [I32, I32, I32, ctypes.POINTER(P)]
    lib.pf_build_network.restype = ctypes.c_int
    lib.pf_build_network_ex.argtypes = [I32, I32, I32] + [P] * 8 + [I32] + [P] * 5 + [I32, I32, I32, I32,
                                                                                ctypes.POINTER(P)]
    lib.pf_build_network_ex.restype = ctypes.c_int
    lib.pf_destroy.argtypes = [P]
    lib.pf_destroy.restype = None
    lib.pf_query.argtypes = [P, ctypes.POINTER(pf_dims)]
    lib.pf_query.restype = ctypes.c_int
    lib.pf_get_structure.argtypes = [P, I32, P]
    lib.pf_get_structure.restype = ctypes.c_int
    lib.pf_last_error.argtypes = [P]
    lib.pf_last_error.restype = ctypes.c_char_p
    lib.pf_build_error.argtypes = []
    lib.pf_build_error.restype = ctypes.c_char_p
    lib.pf_eval_constraints.argtypes = [P, I32] + [P] * 9 + [VP]
    lib.pf_eval_constraints.restype = ctypes.c_int
    lib.pf_jacobian.argtypes = [P, I32, P, P, P, P, P, P, VP]
    lib.pf_jacobian.restype = ctypes.c_int
    lib.pf_reduced_hessian_batch.argtypes = [P, I32] + [P] * 8 + [I32, I32, P, VP]
    lib.pf_reduced_hessian_batch.restype = ctypes.c_int
    lib.pf_condensed_kkt_solve.argtypes = [P, I32, P, P, D, P, I32, P, VP]
    lib.pf_condensed_kkt_solve.restype = ctypes.c_int
    lib.pf_condensed_rhs.argtypes = [P, I32] + [P] * 9 + [VP]
    lib.pf_condensed_rhs.restype = ctypes.c_int
    lib.pf_recover_step.argtypes = [P, I32] + [P] * 10 + [VP]
    lib.pf_recover_step.restype = ctypes.c_int
    lib.pf_power_flow.argtypes = [P, I32] + [P] * 6 + [D, I32, P, P, P, VP]
    lib.pf_power_flow.restype = ctypes.c_int
    lib.pf_reduced_gradient.argtypes = [P, I32] + [P] * 7 + [VP]
    lib.pf_reduced_gradient.restype = ctypes.c_int
    lib.pf_condensed_kkt_solve_reg.argtypes = [P, I32, P, P, D, D, D, D, P, I32, P, P, P, VP]
    lib.pf_condensed_kkt_solve_reg.restype = ctypes.c_int
    lib.pf_launch_count.argtypes = [P]
    lib.pf_launch_count.restype = ctypes.c_int64
    lib.pf_profile.argtypes = [P, I32]
    lib.pf_profile.restype = ctypes.c_int
    lib.pf_kernel_times.argtypes = [P, P, I32]
    lib.pf_kernel_times.restype = ctypes.c_int32
    _lib = lib
    return lib


def _host_ptr(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(ctypes.c_void_p)


def _cplx(a):
    a = np.asarray(a, dtype=np.complex128)
    return np.ascontiguousarray(np.stack([a.real, a.imag], axis=-1).ravel())


def _dev(t, name, dtype=None, numel=None):
    """Pointer of a CUDA tensor (or None)."""
    if t is None:
        return None
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("%s must be a CUDA torch tensor (no CPU fallback)" % name)
    if not t.is_contiguous():
        raise ValueError("%s must be contiguous" % name)
    if dtype is not None and t.dtype != dtype:
        raise TypeError("%s must be %s, got %s" % (name, dtype, t.dtype))
    if numel is not None and t.numel() != numel:
        raise ValueError("%s has %d elements, expected %d" % (name, t.numel(), numel))
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class Network:
    """A built network handle (pf_build_network) plus typed wrappers of the
    compute entry points.  All tensors are CUDA float64 / int32."""

    def __init__(self, net, max_batch, max_scen=1, device=0, tile_cols=0):
        lib = load_library()
        self._lib = lib
        keep = []

        def hp(a, dt):
            arr, p = _host_ptr(a, dt)
            keep.append(arr)
            return p

        def hc(a):
            arr = _cplx(a)
            keep.append(arr)
            return arr.ctypes.data_as(ctypes.c_void_p)

        h = ctypes.c_void_p()
        st = lib.pf_build_network_ex(
            int(net["n_b"]), int(net["n_l"]), int(net["n_g"]),
            hp(net["line_from"], np.int32), hp(net["line_to"], np.int32),
            hc(net["Y_ff"]), hc(net["Y_ft"]), hc(net["Y_tf"]), hc(net["Y_tt"]), hc(net["Y_sh"]),
            hp(net["gen_bus"], np.int32), int(net["ref_bus"]),
            hp(net["p_d"], np.float64), hp(net["q_d"], np.float64), hp(net["F_max"], np.float64),
            hp(net["c_quad"], np.float64), hp(net["c_lin"], np.float64),
            int(max_batch), int(max_scen), int(device), int(tile_cols), ctypes.byref(h))
        if st != PF_OK:
            raise PFError(st, lib.pf_build_error().decode())
        self._h = h
        self.device = device
        d = pf_dims()
        lib.pf_query(h, ctypes.byref(d))
        self.dims = {k: getattr(d, k) for k, _ in pf_dims._fields_}

    def close(self):
        if getattr(self, "_h", None):
            self._lib.pf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st != PF_OK:
            raise PFError(st, "%s: %s" % (what, self._lib.pf_last_error(self._h).decode()))

    def structure(self, name):
        d = self.dims
        sizes = dict(x_theta=d["n_b"], x_v=d["n_b"], u_v=d["n_b"], u_p=d["n_g"], gx_ptr=d["n_x"] + 1,
                     gx_idx=d["nnz_gx"], gu_ptr=d["n_x"] + 1, gu_idx=d["nnz_gu"], a_ptr=d["m"] + 1,
                     a_idx=d["nnz_a"], bus_order=d["n_blocks"], perm=d["n_x"], block_ptr=d["n_blocks"] + 1,
                     lu_ptr=d["n_x"] + 1, lu_idx=d["nnz_lu"], level_l_ptr=d["n_levels_l"] + 1,
                     level_l_blk=d["n_blocks"], level_u_ptr=d["n_levels_u"] + 1, level_u_blk=d["n_blocks"],
                     front_row=d["front_rows"], lu_subtree_ptr=d["lu_pairs"] + 1, lu_level_blk=d["n_blocks"])
        if name == "lu_subtree_blk":
            sizes[name] = int(self.structure("lu_subtree_ptr")[-1])
        out = np.zeros(max(sizes[name], 1), dtype=np.int32)
        self._check(self._lib.pf_get_structure(self._h, STRUCTURE[name], out.ctypes.data_as(ctypes.c_void_p)),
                    "pf_get_structure")
        return out[: sizes[name]]

    def launch_count(self):
        return int(self._lib.pf_launch_count(self._h))

    KERNELS = ("k_fwd", "k_mu", "k_hvp", "k_adj", "k_lu", "k_proj", "k_chol_dag")

    def profile(self, enable=True):
        self._check(self._lib.pf_profile(self._h, int(enable)), "pf_profile")

    def kernel_times(self):
        """Per-kernel ms of the last reduction / jacobian calls (profiling on)."""
        ms = (ctypes.c_float * 7)()
        k = self._lib.pf_kernel_times(self._h, ctypes.cast(ms, ctypes.c_void_p), 7)
        return {self.KERNELS[i]: float(ms[i]) for i in range(k)}

    # ---------------------------------------------------------------- compute
    def pf_eval_constraints(self, n_scen, v, theta, p_g, q_g, p_d=None, q_d=None, G=None, H=None, s_flow=None,
                            stream=None):
        import torch
        d = self.dims
        f64 = torch.float64
        dev = v.device
        if G is None:
            G = torch.empty(n_scen, 2 * d["n_b"], dtype=f64, device=dev)
        st = self._lib.pf_eval_constraints(
            self._h, n_scen, _dev(v, "v", f64, n_scen * d["n_b"]), _dev(theta, "theta", f64, n_scen * d["n_b"]),
            _dev(p_g, "p_g", f64, n_scen * d["n_g"]), _dev(q_g, "q_g", f64, n_scen * d["n_g"]),
            _dev(p_d, "p_d", f64, n_scen * d["n_b"]), _dev(q_d, "q_d", f64, n_scen * d["n_b"]),
            _dev(G, "G", f64, n_scen * 2 * d["n_b"]), _dev(H, "H", f64, n_scen * 2 * d["n_l"]),
            _dev(s_flow, "s_flow", f64, n_scen * 4 * d["n_l"]), _stream(stream))
        self._check(st, "pf_eval_constraints")
        return G, H, s_flow

    def pf_jacobian(self, n_scen, v, theta, Gx_val=None, Gu_val=None, A_val=None, info=None, stream=None):
        import torch
        d = self.dims
        f64 = torch.float64
        st = self._lib.pf_jacobian(
            self._h, n_scen, _dev(v, "v", f64, n_scen * d["n_b"]), _dev(theta, "theta", f64, n_scen * d["n_b"]),
            _dev(Gx_val, "Gx_val", f64, n_scen * d["nnz_gx"]), _dev(Gu_val, "Gu_val", f64, n_scen * d["nnz_gu"]),
            _dev(A_val, "A_val", f64, n_scen * d["nnz_a"]), _dev(info, "info", torch.int32, n_scen),
            _stream(stream))
        self._check(st, "pf_jacobian")
        return Gx_val, Gu_val, A_val, info

    def pf_reduced_hessian_batch(self, n_scen, v, theta, lam, y, KV, sigma_s=None, sigma_x=None, V=None, col0=0,
                                 N=None, p_d=None, stream=None):
        import torch
        d = self.dims
        f64 = torch.float64
        if N is None:
            N = d["n_u"]
        st = self._lib.pf_reduced_hessian_batch(
            self._h, n_scen, _dev(v, "v", f64, n_scen * d["n_b"]), _dev(theta, "theta", f64, n_scen * d["n_b"]),
            _dev(p_d, "p_d", f64, n_scen * d["n_b"]), _dev(lam, "lambda", f64, n_scen * d["n_x"]),
            _dev(y, "y", f64, n_scen * d["m"]), _dev(sigma_s, "sigma_s", f64, n_scen * d["m"]),
            _dev(sigma_x, "sigma_x", f64, n_scen * d["n_x"]), _dev(V, "V", f64, n_scen * N * d["n_u"]),
            int(col0), int(N), _dev(KV, "KV", f64, n_scen * N * d["n_u"]), _stream(stream))
        self._check(st, "pf_reduced_hessian_batch")
        return KV

    def pf_condensed_kkt_solve(self, n_scen, K, sigma_u=None, delta_w=0.0, rhs=None, nrhs=0, info=None,
                               stream=None):
        import torch
        d = self.dims
        f64 = torch.float64
        st = self._lib.pf_condensed_kkt_solve(
            self._h, n_scen, _dev(K, "K", f64, n_scen * d["n_u"] ** 2),
            _dev(sigma_u, "sigma_u", f64, n_scen * d["n_u"]), float(delta_w),
            _dev(rhs, "rhs", f64, n_scen * nrhs * d["n_u"]) if nrhs > 0 else None, int(nrhs),
            _dev(info, "info", torch.int32, n_scen), _stream(stream))
        self._check(st, "pf_condensed_kkt_solve")
        return K, rhs, info

    # ---------------------------------------------------------------- NEXT-1 / NEXT-2
    def kkt_len(self):
        d = self.dims
        return 2 * d["n_x"] + d["n_u"] + 2 * d["m"]

    def pf_condensed_rhs(self, n_scen, v, theta, lam, y, r, b=None, sigma_s=None, sigma_x=None, p_d=None,
                         stream=None):
        import torch
        d = self.dims
        f64 = torch.float64
        if b is None:
            b = torch.empty(n_scen, d["n_u"], dtype=f64, device=r.device)
        st = self._lib.pf_condensed_rhs(
            self._h, n_scen, _dev(v, "v", f64, n_scen * d["n_b"]), _dev(theta, "theta", f64, n_scen * d["n_b"]),
            _dev(p_d, "p_d", f64, n_scen * d["n_b"]), _dev(lam, "lambda", f64, n_scen * d["n_x"]),
            _dev(y, "y", f64, n_scen * d["m"]), _dev(sigma_s, "sigma_s", f64, n_scen * d["m"]),
            _dev(sigma_x, "sigma_x", f64, n_scen * d["n_x"]), _dev(r, "r", f64, n_scen * self.kkt_len()),
            _dev(b, "b", f64, n_scen * d["n_u"]), _stream(stream))
        self._check(st, "pf_condensed_rhs")
        return b

    def pf_recover_step(self, n_scen, v, theta, lam, y, r, p_u, p=None, sigma_s=None, sigma_x=None, p_d=None,
                        stream=None):
        import torch
        d = self.dims
        f64 = torch.float64
        if p is None:
            p = torch.empty(n_scen, self.kkt_len(), dtype=f64, device=r.device)
        st = self._lib.pf_recover_step(
            self._h, n_scen, _dev(v, "v", f64, n_scen * d["n_b"]), _dev(theta, "theta", f64, n_scen * d["n_b"]),
            _dev(p_d, "p_d", f64, n_scen * d["n_b"]), _dev(lam, "lambda", f64, n_scen * d["n_x"]),
            _dev(y, "y", f64, n_scen * d["m"]), _dev(sigma_s, "sigma_s", f64, n_scen * d["m"]),
            _dev(sigma_x, "sigma_x", f64, n_scen * d["n_x"]), _dev(r, "r", f64, n_scen * self.kkt_len()),
            _dev(p_u, "p_u", f64, n_scen * d["n_u"]), _dev(p, "p", f64, n_scen * self.kkt_len()), _stream(stream))
        self._check(st, "pf_recover_step")
        return p

    def pf_power_flow(self, n_scen, v, theta, p_g, q_g=None, p_d=None, q_d=None, tol=1e-10, max_iter=20,
                      stream=None):
        """Newton power flow in place on (v, theta); returns (iters, resid, info) host arrays."""
        import torch
        d = self.dims
        f64 = torch.float64
        iters = np.zeros(n_scen, dtype=np.int32)
        resid = np.zeros(n_scen, dtype=np.float64)
        info = np.zeros(n_scen, dtype=np.int32)
        st = self._lib.pf_power_flow(
            self._h, n_scen, _dev(v, "v", f64, n_scen * d["n_b"]), _dev(theta, "theta", f64, n_scen * d["n_b"]),
            _dev(p_g, "p_g", f64, n_scen * d["n_g"]), _dev(q_g, "q_g", f64, n_scen * d["n_g"]),
            _dev(p_d, "p_d", f64, n_scen * d["n_b"]), _dev(q_d, "q_d", f64, n_scen * d["n_b"]), float(tol),
            int(max_iter), iters.ctypes.data_as(ctypes.c_void_p), resid.ctypes.data_as(ctypes.c_void_p),
            info.ctypes.data_as(ctypes.c_void_p), _stream(stream))
        self._check(st, "pf_power_flow")
        return iters, resid, info

    def pf_reduced_gradient(self, n_scen, v, theta, p_g, y, lam=None, grad=None, p_d=None, stream=None):
        import torch
        d = self.dims
        f64 = torch.float64
        if grad is None:
            grad = torch.empty(n_scen, d["n_u"], dtype=f64, device=y.device)
        st = self._lib.pf_reduced_gradient(
            self._h, n_scen, _dev(v, "v", f64, n_scen * d["n_b"]), _dev(theta, "theta", f64, n_scen * d["n_b"]),
            _dev(p_g, "p_g", f64, n_scen * d["n_g"]), _dev(p_d, "p_d", f64, n_scen * d["n_b"]),
            _dev(y, "y", f64, n_scen * d["m"]), _dev(lam, "lambda", f64, n_scen * d["n_x"]),
            _dev(grad, "grad", f64, n_scen * d["n_u"]), _stream(stream))
        self._check(st, "pf_reduced_gradient")
        return lam, grad

    # ---------------------------------------------------------------- NEXT-3
    def pf_condensed_kkt_solve_reg(self, n_scen, K, sigma_u=None, delta_init=0.0, delta_first=1e-8, growth=10.0,
                                   delta_max=1e12, rhs=None, nrhs=0, stream=None):
        """Regularized condensed solve; returns (delta, trials, info) host arrays."""
        import torch
        d = self.dims
        f64 = torch.float64
        delta = np.zeros(n_scen, dtype=np.float64)
        trials = np.zeros(n_scen, dtype=np.int32)
        info = np.zeros(n_scen, dtype=np.int32)
        st = self._lib.pf_condensed_kkt_solve_reg(
            self._h, n_scen, _dev(K, "K", f64, n_scen * d["n_u"] ** 2), _dev(sigma_u, "sigma_u", f64, n_scen * d["n_u"]),
            float(delta_init), float(delta_first), float(growth), float(delta_max),
            _dev(rhs, "rhs", f64, n_scen * nrhs * d["n_u"]) if nrhs > 0 else None, int(nrhs),
            delta.ctypes.data_as(ctypes.c_void_p), trials.ctypes.data_as(ctypes.c_void_p),
            info.ctypes.data_as(ctypes.c_void_p), _stream(stream))
        self._check(st, "pf_condensed_kkt_solve_reg")
        return delta, trials, info
