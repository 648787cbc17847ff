"""CPU oracle for the AIDW hot path — TEST INFRASTRUCTURE ONLY.

Two libraries, both loaded through ctypes:

* ``liborc``    — ``oracle/aidw_oracle.c``, a plain-C restatement of the
  reference algorithm (each function cites proj/include/aidw/<file>:<lines>).
* ``libaidw_ref`` — the reference itself, compiled in place from
  /root/reference/proj/include by ``oracle/Makefile`` (target ``ref``) into
  ``oracle/_ref/``.  Present wherever ``__graft_entry__.build()`` ran with the
  reference mounted; the .so travels to the GPU box with the repo snapshot.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product
(``paper_1601_05904_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "_build", "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libaidw_ref.so")

_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)
_szp = C.POINTER(C.c_size_t)


def _p(a, t):
    return a.ctypes.data_as(t)


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, code, message="", index=-1):
        super().__init__(f"oracle error code={code} index={index} {message}")
        self.code = code
        self.index = index
        self.message = message


class GridConfigC(C.Structure):
    _fields_ = [("cell_width", C.c_double), ("n_col", C.c_int), ("n_row", C.c_int),
                ("min_x", C.c_double), ("min_y", C.c_double)]


def build_oracle(quiet=True):
    """Compile liborc.so (gcc -ffp-contract=off) if missing or stale."""
    src = os.path.join(HERE, "aidw_oracle.c")
    if os.path.exists(ORC_PATH) and os.path.getmtime(ORC_PATH) >= os.path.getmtime(src):
        return ORC_PATH
    import subprocess
    subprocess.run(["make", "-C", HERE, "all"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)
    return ORC_PATH


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        build_oracle()
        _orc = C.CDLL(ORC_PATH)
        _orc.orc_dist_sq.restype = C.c_double
    return _orc


def ref_available():
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_PATH} not built (make -C oracle ref)")
        _ref = C.CDLL(REF_PATH)
        _ref.ref_normalize_mu.restype = C.c_double
        _ref.ref_normalize_mu.argtypes = [C.c_double] * 3
    return _ref


def _check(rc, idx=-1, msg=b""):
    if rc != 0:
        raise OracleError(rc, msg.decode() if isinstance(msg, bytes) else str(msg), idx)


# ---------------------------------------------------------------- generators
def generate_points(count, bbox=(0.0, 0.0, 1.0, 1.0), seed=42, rule=0):
    xs, ys, zs = (np.empty(count) for _ in range(3))
    _check(orc().orc_generate_points(C.c_size_t(count), *(C.c_double(v) for v in bbox),
                                     C.c_uint64(seed), C.c_int(rule), _p(xs, _dp), _p(ys, _dp),
                                     _p(zs, _dp)))
    return xs, ys, zs


def generate_queries(count, bbox=(0.0, 0.0, 1.0, 1.0), seed=43):
    xs, ys = np.empty(count), np.empty(count)
    _check(orc().orc_generate_queries(C.c_size_t(count), *(C.c_double(v) for v in bbox),
                                      C.c_uint64(seed), _p(xs, _dp), _p(ys, _dp)))
    return xs, ys


def generate_clustered(count, blobs=20, sigma=0.03, center_seed=5, seed=42, with_values=True):
    xs, ys, zs = np.empty(count), np.empty(count), np.zeros(count)
    _check(orc().orc_generate_clustered(C.c_size_t(count), C.c_int(blobs), C.c_double(sigma),
                                        C.c_uint64(center_seed), C.c_uint64(seed),
                                        C.c_int(1 if with_values else 0), _p(xs, _dp),
                                        _p(ys, _dp), _p(zs, _dp)))
    return (xs, ys, zs) if with_values else (xs, ys)


# ---------------------------------------------------------------- geometry
def compute_bbox(dx, dy, qx=None, qy=None):
    dx, dy = _d(dx), _d(dy)
    qx = _d(qx if qx is not None else []); qy = _d(qy if qy is not None else [])
    out = np.empty(4)
    _check(orc().orc_compute_bbox(_p(dx, _dp), _p(dy, _dp), C.c_size_t(dx.size), _p(qx, _dp),
                                  _p(qy, _dp), C.c_size_t(qx.size), _p(out, _dp)))
    return out


def choose_cell_width(m, bbox, factor=4.0):
    out = C.c_double()
    bb = _d(bbox)
    _check(orc().orc_choose_cell_width(C.c_size_t(m), _p(bb, _dp), C.c_double(factor),
                                       C.byref(out)))
    return out.value


def make_grid_config(bbox, cell_width):
    cfg = GridConfigC()
    bb = _d(bbox)
    _check(orc().orc_make_grid_config(_p(bb, _dp), C.c_double(cell_width), C.byref(cfg)))
    return cfg


def grid_config(cell_width, n_col, n_row, min_x=0.0, min_y=0.0):
    return GridConfigC(cell_width, n_col, n_row, min_x, min_y)


def locate_cell(x, y, cfg):
    col, row = C.c_int(), C.c_int()
    _check(orc().orc_locate_cell(C.c_double(x), C.c_double(y), C.byref(cfg), C.byref(col),
                                 C.byref(row)))
    return col.value, row.value


def build_index(xs, ys, cfg):
    xs, ys = _d(xs), _d(ys)
    m = xs.size
    cells = cfg.n_col * cfg.n_row
    ids = np.empty(m, np.uint32)
    cs = np.empty(cells + 1, np.uint32)
    sx, sy = np.empty(m), np.empty(m)
    fail = C.c_int64(-1)
    _check(orc().orc_build_index(_p(xs, _dp), _p(ys, _dp), C.c_size_t(m), C.byref(cfg),
                                 _p(ids, _u32p), _p(cs, _u32p), _p(sx, _dp), _p(sy, _dp),
                                 C.byref(fail)), fail.value)
    return ids, cs, sx, sy


def dist_sq(qx, qy, px, py):
    return orc().orc_dist_sq(C.c_double(qx), C.c_double(qy), C.c_double(px), C.c_double(py))


# ---------------------------------------------------------------- kNN
def knn_grid(qx, qy, cfg, grid, m, k):
    """Batch grid kNN.  Returns (d2[n,k], ids[n,k], avg[n], exhausted[n])."""
    qx, qy = _d(qx), _d(qy)
    n = qx.size
    ids_s, cs, sx, sy = grid
    d2 = np.empty((n, k)); idn = np.empty((n, k), np.uint32)
    avg = np.empty(n); exh = np.zeros(n, np.int32)
    fail = C.c_int64(-1)
    _check(orc().orc_knn_stage_grid(_p(qx, _dp), _p(qy, _dp), C.c_size_t(n), C.byref(cfg),
                                    _p(cs, _u32p), _p(ids_s, _u32p), _p(sx, _dp), _p(sy, _dp),
                                    C.c_size_t(m), C.c_int(k), _p(d2, _dp), _p(idn, _u32p),
                                    _p(avg, _dp), _p(exh, _ip), C.byref(fail)), fail.value)
    return d2, idn, avg, exh.astype(bool)


def knn_brute(qx, qy, xs, ys, k):
    qx, qy, xs, ys = _d(qx), _d(qy), _d(xs), _d(ys)
    n = qx.size
    d2 = np.empty((n, k)); idn = np.empty((n, k), np.uint32); avg = np.empty(n)
    fail = C.c_int64(-1)
    _check(orc().orc_knn_stage_brute(_p(qx, _dp), _p(qy, _dp), C.c_size_t(n), _p(xs, _dp),
                                     _p(ys, _dp), C.c_size_t(xs.size), C.c_int(k), _p(d2, _dp),
                                     _p(idn, _u32p), _p(avg, _dp), C.byref(fail)), fail.value)
    return d2, idn, avg


# ---------------------------------------------------------------- adaptive
def adaptive_alpha(r_obs, m, area, k=15, r_min=0.0, r_max=2.0,
                   levels=(0.5, 1.0, 2.0, 3.0, 4.0), list_len=None, exhausted=False):
    rec = np.empty(5)
    lv = _d(levels)
    _check(orc().orc_adaptive_alpha(C.c_double(r_obs), C.c_size_t(k if list_len is None else list_len),
                                    C.c_int(int(exhausted)), C.c_size_t(m), C.c_double(area),
                                    C.c_int(k), C.c_double(r_min), C.c_double(r_max),
                                    _p(lv, _dp), _p(rec, _dp)))
    return rec


def normalize_mu(R, r_min=0.0, r_max=2.0):
    out = C.c_double()
    _check(orc().orc_normalize_mu(C.c_double(R), C.c_double(r_min), C.c_double(r_max),
                                  C.byref(out)))
    return out.value


def alpha_from_mu(mu, levels=(0.5, 1.0, 2.0, 3.0, 4.0)):
    out = C.c_double()
    lv = _d(levels)
    _check(orc().orc_alpha_from_mu(C.c_double(mu), _p(lv, _dp), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- weighting
def predict_with_alphas(qx, qy, xs, ys, zs, alphas, variant=0):
    qx, qy, xs, ys, zs, al = _d(qx), _d(qy), _d(xs), _d(ys), _d(zs), _d(alphas)
    pred = np.empty(qx.size)
    _check(orc().orc_predict_with_alphas(_p(qx, _dp), _p(qy, _dp), C.c_size_t(qx.size),
                                         _p(xs, _dp), _p(ys, _dp), _p(zs, _dp),
                                         C.c_size_t(xs.size), _p(al, _dp), C.c_int(variant),
                                         _p(pred, _dp)))
    return pred


def aidw_predict_all(qx, qy, xs, ys, zs, r_obs, k=15, r_min=0.0, r_max=2.0,
                     levels=(0.5, 1.0, 2.0, 3.0, 4.0), area=0.0, variant=0, list_len=None,
                     exhausted=None):
    qx, qy, xs, ys, zs, ro = _d(qx), _d(qy), _d(xs), _d(ys), _d(zs), _d(r_obs)
    n = qx.size
    ll = np.full(n, k, np.uintp) if list_len is None else np.ascontiguousarray(list_len, np.uintp)
    ex = np.zeros(n, np.int32) if exhausted is None else np.ascontiguousarray(exhausted, np.int32)
    lv = _d(levels)
    pred, al = np.empty(n), np.empty(n)
    fail = C.c_int64(-1)
    _check(orc().orc_aidw_predict_all(_p(qx, _dp), _p(qy, _dp), C.c_size_t(n), _p(xs, _dp),
                                      _p(ys, _dp), _p(zs, _dp), C.c_size_t(xs.size), _p(ro, _dp),
                                      _p(ll, _szp), _p(ex, _ip), C.c_int(k), C.c_double(r_min),
                                      C.c_double(r_max), _p(lv, _dp), C.c_double(area),
                                      C.c_int(variant), _p(pred, _dp), _p(al, _dp),
                                      C.byref(fail)), fail.value)
    return pred, al


def pipeline(dx, dy, dz, qx, qy, k=10, factor=4.0, variant=0, r_min=0.0, r_max=2.0,
             levels=(0.5, 1.0, 2.0, 3.0, 4.0), area=0.0):
    """Oracle run_pipeline (aidw mode, grid engine): returns a dict."""
    dx, dy, dz, qx, qy = _d(dx), _d(dy), _d(dz), _d(qx), _d(qy)
    m = dx.size
    k = min(k, m)
    bb = compute_bbox(dx, dy, qx, qy)
    cfg = make_grid_config(bb, choose_cell_width(m, bb, factor))
    grid = build_index(dx, dy, cfg)
    d2, ids, avg, exh = knn_grid(qx, qy, cfg, grid, m, k)
    pred, al = aidw_predict_all(qx, qy, dx, dy, dz, avg, k=k, r_min=r_min, r_max=r_max,
                                levels=levels, area=area, variant=variant,
                                list_len=np.full(qx.size, min(k, m)), exhausted=exh)
    return dict(cfg=cfg, grid=grid, d2=d2, ids=ids, avg=avg, exhausted=exh, pred=pred,
                alpha=al, bbox=bb)


# ---------------------------------------------------------------- reference (.so)
_MSG = 512


def _msg():
    return C.create_string_buffer(_MSG)


def ref_generate_points(count, bbox=(0.0, 0.0, 1.0, 1.0), seed=42, rule=0):
    xs, ys, zs = (np.empty(count) for _ in range(3))
    bb = _d(bbox); m = _msg()
    _check(ref().ref_generate_points(C.c_size_t(count), _p(bb, _dp), C.c_uint64(seed),
                                     C.c_int(rule), _p(xs, _dp), _p(ys, _dp), _p(zs, _dp), m,
                                     C.c_size_t(_MSG)), -1, m.value)
    return xs, ys, zs


def ref_generate_queries(count, bbox=(0.0, 0.0, 1.0, 1.0), seed=43):
    xs, ys = np.empty(count), np.empty(count)
    bb = _d(bbox); m = _msg()
    _check(ref().ref_generate_queries(C.c_size_t(count), _p(bb, _dp), C.c_uint64(seed),
                                      _p(xs, _dp), _p(ys, _dp), m, C.c_size_t(_MSG)), -1, m.value)
    return xs, ys


def ref_grid_config(dx, dy, qx, qy, factor=4.0):
    dx, dy, qx, qy = _d(dx), _d(dy), _d(qx), _d(qy)
    out = np.empty(5); m = _msg()
    _check(ref().ref_grid_config(_p(dx, _dp), _p(dy, _dp), C.c_size_t(dx.size), _p(qx, _dp),
                                 _p(qy, _dp), C.c_size_t(qx.size), C.c_double(factor),
                                 _p(out, _dp), m, C.c_size_t(_MSG)), -1, m.value)
    return out


def ref_build_index(xs, ys, cfg5):
    xs, ys, c = _d(xs), _d(ys), _d(cfg5)
    mm = xs.size
    cells = int(c[1]) * int(c[2])
    ids = np.empty(mm, np.uint32); cs = np.empty(cells + 1, np.uint32)
    sx, sy = np.empty(mm), np.empty(mm); m = _msg()
    _check(ref().ref_build_index(_p(xs, _dp), _p(ys, _dp), C.c_size_t(mm), _p(c, _dp),
                                 _p(ids, _u32p), _p(cs, _u32p), _p(sx, _dp), _p(sy, _dp), m,
                                 C.c_size_t(_MSG)), -1, m.value)
    return ids, cs, sx, sy


def ref_knn_stage(qx, qy, dx, dy, k, engine=0, factor=4.0, workers=1):
    qx, qy, dx, dy = _d(qx), _d(qy), _d(dx), _d(dy)
    n = qx.size
    d2 = np.empty((n, k)); avg = np.empty(n); exh = np.zeros(n, np.int32)
    lens = np.empty(n, np.int64); m = _msg()
    _check(ref().ref_knn_stage(_p(qx, _dp), _p(qy, _dp), C.c_size_t(n), _p(dx, _dp), _p(dy, _dp),
                               C.c_size_t(dx.size), C.c_int(k), C.c_int(engine),
                               C.c_double(factor), C.c_int(workers), _p(d2, _dp), _p(avg, _dp),
                               _p(exh, _ip), _p(lens, _i64p), m, C.c_size_t(_MSG)), -1, m.value)
    return d2, avg, exh.astype(bool), lens


def ref_adaptive_alpha(r_obs, m, area, k=15, r_min=0.0, r_max=2.0,
                       levels=(0.5, 1.0, 2.0, 3.0, 4.0), list_len=None, exhausted=False):
    rec = np.empty(5); lv = _d(levels); msg = _msg()
    _check(ref().ref_adaptive_alpha(C.c_double(r_obs), C.c_size_t(k if list_len is None else list_len),
                                    C.c_int(int(exhausted)), C.c_size_t(m), C.c_double(area),
                                    C.c_int(k), C.c_double(r_min), C.c_double(r_max),
                                    _p(lv, _dp), _p(rec, _dp), msg, C.c_size_t(_MSG)), -1,
           msg.value)
    return rec


def ref_predict_all(dx, dy, dz, qx, qy, mode=1, engine=0, variant=1, pinned=False, k=15,
                    r_min=0.0, r_max=2.0, levels=(0.5, 1.0, 2.0, 3.0, 4.0), area=0.0,
                    alpha=2.0, factor=4.0, workers=1):
    dx, dy, dz, qx, qy = _d(dx), _d(dy), _d(dz), _d(qx), _d(qy)
    n = qx.size
    pred, al = np.empty(n), np.empty(n); lv = _d(levels); m = _msg()
    _check(ref().ref_predict_all(_p(dx, _dp), _p(dy, _dp), _p(dz, _dp), C.c_size_t(dx.size),
                                 _p(qx, _dp), _p(qy, _dp), C.c_size_t(n), C.c_int(mode),
                                 C.c_int(engine), C.c_int(variant), C.c_int(int(pinned)),
                                 C.c_int(k), C.c_double(r_min), C.c_double(r_max), _p(lv, _dp),
                                 C.c_double(area), C.c_double(alpha), C.c_double(factor),
                                 C.c_int(workers), _p(pred, _dp), _p(al, _dp), m,
                                 C.c_size_t(_MSG)), -1, m.value)
    return pred, al


def ref_run_pipeline(dx, dy, dz, qx, qy, mode=1, engine=0, variant=1, k=15, r_min=0.0,
                     r_max=2.0, levels=(0.5, 1.0, 2.0, 3.0, 4.0), area=0.0, alpha=2.0,
                     factor=4.0, workers=0):
    """Reference cli::run_pipeline; returns (pred, alphas, timings_ms[4], k_eff)."""
    dx, dy, dz, qx, qy = _d(dx), _d(dy), _d(dz), _d(qx), _d(qy)
    n = qx.size
    pred, al, tm = np.empty(n), np.empty(n), np.empty(4)
    keff = C.c_int(); lv = _d(levels); m = _msg()
    _check(ref().ref_run_pipeline(_p(dx, _dp), _p(dy, _dp), _p(dz, _dp), C.c_size_t(dx.size),
                                  _p(qx, _dp), _p(qy, _dp), C.c_size_t(n), C.c_int(mode),
                                  C.c_int(engine), C.c_int(variant), C.c_int(k),
                                  C.c_double(r_min), C.c_double(r_max), _p(lv, _dp),
                                  C.c_double(area), C.c_double(alpha), C.c_double(factor),
                                  C.c_int(workers), _p(pred, _dp), _p(al, _dp), _p(tm, _dp),
                                  C.byref(keff), m, C.c_size_t(_MSG)), -1, m.value)
    return pred, al, tm, keff.value


def ref_hardware_threads():
    return int(ref().ref_hardware_threads())


def raster_lattice(nx, ny, bbox):
    """cmd_raster lattice (cli.hpp:495-507), C restatement."""
    xs, ys = np.empty(nx * ny), np.empty(nx * ny)
    bb = _d(bbox)
    _check(orc().orc_raster_lattice(C.c_size_t(nx), C.c_size_t(ny), _p(bb, _dp), _p(xs, _dp),
                                    _p(ys, _dp)))
    return xs, ys


def ref_cmd_raster(dx, dy, dz, nx, ny, k=15, workers=0, tmpdir="/tmp"):
    """The reference's own cli::cmd_raster (data written to CSV by the
    reference writer, read back by its parser, raster written by its
    write_raster_asc).  Returns (values (nrows*ncols,), meta dict, asc path)."""
    import os
    dx, dy, dz = _d(dx), _d(dy), _d(dz)
    csv = os.path.join(tmpdir, f"aidw_ref_raster_{os.getpid()}.csv").encode()
    asc = os.path.join(tmpdir, f"aidw_ref_raster_{os.getpid()}.asc").encode()
    vals, meta = np.empty(nx * ny), np.empty(5)
    m = _msg()
    _check(ref().ref_cmd_raster(_p(dx, _dp), _p(dy, _dp), _p(dz, _dp), C.c_size_t(dx.size),
                                C.c_size_t(nx), C.c_size_t(ny), C.c_int(k), C.c_int(workers), csv,
                                asc, _p(vals, _dp), _p(meta, _dp), m, C.c_size_t(_MSG)), -1,
           m.value)
    return vals, dict(zip(("ncols", "nrows", "xllcorner", "yllcorner", "cellsize"), meta)), \
        asc.decode()


def ref_read_points_csv(path, with_values=True, cap=1 << 22):
    """The reference's read_data_csv / read_query_csv.  Returns (xs, ys, zs)
    or raises OracleError(code, message)."""
    xs, ys, zs = np.empty(cap), np.empty(cap), np.empty(cap)
    count = C.c_size_t()
    m = _msg()
    rc = ref().ref_read_points_csv(path.encode(), C.c_int(1 if with_values else 0),
                                   C.c_size_t(cap), _p(xs, _dp), _p(ys, _dp), _p(zs, _dp),
                                   C.byref(count), m, C.c_size_t(_MSG))
    if rc != 0:
        raise OracleError(rc, m.value.decode(), -1)
    n = count.value
    return xs[:n].copy(), ys[:n].copy(), (zs[:n].copy() if with_values else None)
