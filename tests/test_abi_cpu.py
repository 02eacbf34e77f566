"""Host-side checks of the C ABI (no GPU needed): the library loads, exports
every symbol include/dmv3d.h declares, and rejects bad arguments with the
documented status before touching the device."""
import ctypes as ct
import os
import re

import numpy as np
import pytest

from paper_2605_18052_b200 import _abi, schedule
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dmv3d.h")).read()
    return sorted(set(re.findall(r"\b(dmv3d_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _abi.lib()
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s
    assert set(_abi.EXPORTED) <= set(syms)
    assert b"sm_100a" in L.dmv3d_version()


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_abi.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def _valid_structs(keep):
    intr = np.zeros((1, 4), np.float32)
    c2w = np.zeros((1, 3, 4), np.float32)
    tp = np.zeros((3, 4, 4, 8), np.float32)
    keep += [intr, c2w, tp]
    cams = _abi.Cameras(1, 4, 4, intr.ctypes.data, c2w.ctypes.data)
    t = _abi.Triplane(4, 8, _abi.F32, tp.ctypes.data, (ct.c_float * 3)(-1, -1, -1),
                      (ct.c_float * 3)(1, 1, 1))
    ws = [np.zeros((16, 8), np.float32), np.zeros((4, 16), np.float32)]
    bs = [np.zeros(16, np.float32), np.zeros(4, np.float32)]
    keep += ws + bs
    warr = (ct.c_void_p * 2)(*[w.ctypes.data for w in ws])
    barr = (ct.c_void_p * 2)(*[b.ctypes.data for b in bs])
    keep += [warr, barr]
    m = _abi.MLP(2, 8, 16, _abi.F32, ct.cast(warr, ct.POINTER(ct.c_void_p)),
                 ct.cast(barr, ct.POINTER(ct.c_void_p)), 0, 0.0, 0.0)
    o = _abi.RenderOpts(16, 0, 0, 0, (ct.c_float * 3)(1, 1, 1), 0.0, -1, -1, 0, None)
    return t, cams, m, o


@pytest.mark.parametrize("mutate,status", [
    (lambda t, c, m, o: setattr(c, "num_views", 0), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: setattr(t, "res", 1), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: setattr(t, "channels", 6), _abi.ERR_UNSUPPORTED),
    (lambda t, c, m, o: setattr(m, "num_layers", 1), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: setattr(m, "num_layers", 9), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: setattr(m, "in_dim", 4), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: setattr(o, "samples_per_ray", 0), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: setattr(o, "samples_per_ray", 1025), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: setattr(o, "term_eps", 1.5), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: (setattr(o, "ray_begin", 5), setattr(o, "ray_end", 4)), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: (setattr(o, "ray_begin", 0), setattr(o, "ray_end", 17)), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: setattr(t, "data", t.data + 4), _abi.ERR_ALIGNMENT),
    (lambda t, c, m, o: setattr(c, "c2w", c.c2w + 8), _abi.ERR_ALIGNMENT),
    (lambda t, c, m, o: setattr(o, "engine", _abi.ENGINE_TCGEN05), _abi.ERR_UNSUPPORTED),
    (lambda t, c, m, o: setattr(m, "hidden", 17), _abi.ERR_UNSUPPORTED),
    (lambda t, c, m, o: setattr(t, "sample_mode", 2), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: setattr(t, "dtype", 3), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: (setattr(o, "tile_size", 6), setattr(o, "tile_count", 2)), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: (setattr(o, "tile_size", 16), setattr(o, "tile_rank", 2),
                         setattr(o, "tile_count", 2)), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: setattr(o, "agg", 3), _abi.ERR_INVALID_ARG),
    (lambda t, c, m, o: setattr(o, "agg", _abi.AGG_CONCAT), _abi.ERR_INVALID_ARG),  # in_dim != 3C
    (lambda t, c, m, o: (setattr(o, "agg", _abi.AGG_CONCAT), setattr(m, "in_dim", 24),
                         setattr(m, "hidden", 32)), _abi.ERR_UNSUPPORTED),  # no (24, 32) concat kernel
])
def test_render_argument_validation(mutate, status):
    keep = []
    t, c, m, o = _valid_structs(keep)
    mutate(t, c, m, o)
    rgb = np.zeros(64, np.float32)
    st = _abi.lib().dmv3d_render_views(ct.byref(t), ct.byref(c), ct.byref(m), ct.byref(o),
                                       rgb.ctypes.data, None, None)
    assert st == status, _abi.lib().dmv3d_last_error()
    assert len(_abi.lib().dmv3d_last_error()) > 0


def test_render_null_rgb_rejected():
    keep = []
    t, c, m, o = _valid_structs(keep)
    st = _abi.lib().dmv3d_render_views(ct.byref(t), ct.byref(c), ct.byref(m), ct.byref(o), None,
                                       None, None)
    assert st == _abi.ERR_INVALID_ARG


@pytest.mark.parametrize("field,value", [("t", 1000), ("t", -1), ("t_prev", 980), ("eta", 1.5)])
def test_ddim_argument_validation(field, value):
    ab = schedule.cosine_alpha_bar()
    d = _abi.DdimParams(ab.ctypes.data_as(ct.POINTER(ct.c_double)), 1000, 980, 960, 0.0, 2.0, -1.0,
                        None, 1)
    setattr(d, field, value)
    x = np.zeros(48, np.float32)
    st = _abi.lib().dmv3d_ddim_step(ct.byref(d), 1, 4, 4, x.ctypes.data, x.ctypes.data, None,
                                    x.ctypes.data, None)
    assert st == _abi.ERR_INVALID_ARG


def test_ddim_eta_needs_z():
    ab = schedule.cosine_alpha_bar()
    d = _abi.DdimParams(ab.ctypes.data_as(ct.POINTER(ct.c_double)), 1000, 980, 960, 0.5, 2.0, -1.0,
                        None, 1)
    x = np.zeros(48, np.float32)
    st = _abi.lib().dmv3d_ddim_step(ct.byref(d), 1, 4, 4, x.ctypes.data, x.ctypes.data, None,
                                    x.ctypes.data, None)
    assert st == _abi.ERR_INVALID_ARG
    assert b"z" in _abi.lib().dmv3d_last_error()


def test_product_schedule_matches_oracle():
    """Host logic: the product's alpha_bar table equals the (pinned) oracle's."""
    assert np.max(np.abs(schedule.cosine_alpha_bar() - oracle.cosine_alpha_bar())) < 1e-14
    ts = schedule.ddim_timesteps()
    assert ts[0] == 980 and ts[-1] == 0 and len(ts) == 50
    assert schedule.ddim_pairs()[-1] == (0, -1)


def test_struct_layout_matches_header(tmp_path):
    """The ctypes mirrors in _abi have the size and field offsets the C compiler gives
    the structs of include/dmv3d.h (gcc, host ABI)."""
    structs = {"dmv3d_cameras": _abi.Cameras, "dmv3d_triplane": _abi.Triplane,
               "dmv3d_mlp": _abi.MLP, "dmv3d_render_opts": _abi.RenderOpts,
               "dmv3d_ddim_params": _abi.DdimParams}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "dmv3d.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f in py._fields_:
            lines.append(f'printf("{cname} {f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines += ["return 0; }"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    r = os.system(f"gcc -I{os.path.join(ROOT, 'include')} {src} -o {exe}")
    assert r == 0
    got = {}
    for ln in os.popen(str(exe)).read().splitlines():
        name, field, val = ln.split()
        got[(name, field)] = int(val)
    for cname, py in structs.items():
        assert got[(cname, "size")] == ct.sizeof(py), cname
        for f in py._fields_:
            assert got[(cname, f[0])] == getattr(py, f[0]).offset, (cname, f[0])


def test_render_validation_fuzz():
    """Random out-of-range mutations of valid arguments always come back as a documented
    error status with a message -- never a crash, never OK -- before any device work."""
    from hypothesis import given, settings, strategies as st

    fields = {
        ("t", "res"): st.integers(-3, 10000), ("t", "channels"): st.integers(-3, 300),
        ("t", "sample_mode"): st.integers(-2, 3), ("t", "dtype"): st.integers(-1, 3),
        ("m", "num_layers"): st.integers(-1, 12), ("m", "in_dim"): st.integers(-1, 300),
        ("m", "hidden"): st.integers(-1, 300), ("m", "hidden_act"): st.integers(-1, 4),
        ("c", "num_views"): st.integers(-1, 8), ("c", "height"): st.integers(-1, 8),
        ("o", "samples_per_ray"): st.integers(-1, 2000), ("o", "agg"): st.integers(-1, 4),
        ("o", "engine"): st.integers(-1, 4), ("o", "term_eps"): st.floats(-1.0, 2.0),
        ("o", "num_peers"): st.integers(-1, 9),
    }
    valid_range = {"res": (2, 8192), "sample_mode": (0, 1), "dtype": (0, 1),
                   "num_layers": (2, 8), "hidden_act": (0, 2), "num_views": (1, 1 << 30),
                   "height": (1, 1 << 30), "samples_per_ray": (1, 1024), "agg": (0, 2),
                   "engine": (0, 2), "num_peers": (0, 7), "channels": (1, 1 << 30)}
    documented = {_abi.OK, _abi.ERR_INVALID_ARG, _abi.ERR_UNSUPPORTED, _abi.ERR_CUDA,
                  _abi.ERR_ALIGNMENT}

    @settings(max_examples=300, deadline=None)
    @given(st.lists(st.sampled_from(sorted(fields)), min_size=1, max_size=3, unique=True), st.data())
    def run(keys, data):
        keep = []
        t, c, m, o = _valid_structs(keep)
        objs = {"t": t, "c": c, "m": m, "o": o}
        out_of_range = False
        for k in keys:
            v = data.draw(fields[k])
            setattr(objs[k[0]], k[1], v)
            lo, hi = valid_range.get(k[1], (-1e30, 1e30))
            if k[1] == "term_eps":
                lo, hi = 0.0, 0.999999
            out_of_range |= not (lo <= v <= hi)
        if not out_of_range:
            return  # a valid call would launch on host pointers: only invalid ones are sent
        rgb = np.zeros(64, np.float32)
        s = _abi.lib().dmv3d_render_views(ct.byref(t), ct.byref(c), ct.byref(m), ct.byref(o),
                                          rgb.ctypes.data, None, None)
        assert s in documented and s != _abi.OK
        assert len(_abi.lib().dmv3d_last_error()) > 0

    run()


def test_select_engine_on_the_host():
    """dmv3d_select_engine resolves AUTO without device work: fp32 storage -> SIMT; bf16
    triplane + weights with hidden 64 and a workspace -> TCGEN05; an explicit TCGEN05
    request the tensor cores cannot serve -> UNSUPPORTED (every documented activation
    is accepted by the tensor-core engine's forward)."""
    keep = []
    t, c, m, o = _valid_structs(keep)
    e = ct.c_int32(-1)
    L = _abi.lib()
    assert L.dmv3d_select_engine(ct.byref(t), ct.byref(m), ct.byref(o), 1, ct.byref(e)) == _abi.OK
    assert e.value == _abi.ENGINE_SIMT
    # a bf16 80-channel triplane with the paper's 80-64-64-64-4 MLP
    tp = np.zeros((3, 4, 4, 80), np.uint16)
    ws = [np.zeros((64, 80), np.uint16), np.zeros((64, 64), np.uint16), np.zeros((64, 64), np.uint16),
          np.zeros((4, 64), np.uint16)]
    bs = [np.zeros(64, np.float32)] * 3 + [np.zeros(4, np.float32)]
    warr = (ct.c_void_p * 4)(*[w.ctypes.data for w in ws])
    barr = (ct.c_void_p * 4)(*[b.ctypes.data for b in bs])
    keep += [tp, ws, bs, warr, barr]
    t2 = _abi.Triplane(4, 80, _abi.BF16, tp.ctypes.data, (ct.c_float * 3)(-1, -1, -1),
                       (ct.c_float * 3)(1, 1, 1))
    nbytes = 0
    for act in (0, 1, 2):
        m2 = _abi.MLP(4, 80, 64, _abi.BF16, ct.cast(warr, ct.POINTER(ct.c_void_p)),
                      ct.cast(barr, ct.POINTER(ct.c_void_p)), act, 0.0, 0.0)
        nbytes = L.dmv3d_workspace_bytes(ct.byref(t2), ct.byref(m2))
        ws_buf = np.zeros(nbytes + 512, np.uint8)
        keep.append(ws_buf)
        o2 = _abi.RenderOpts(16, 0, 0, 0, (ct.c_float * 3)(1, 1, 1), 0.0, -1, -1, 0, None)
        o2.workspace = (ws_buf.ctypes.data + 255) // 256 * 256
        o2.workspace_bytes = nbytes
        assert L.dmv3d_select_engine(ct.byref(t2), ct.byref(m2), ct.byref(o2), 1, ct.byref(e)) == _abi.OK
        assert e.value == _abi.ENGINE_TCGEN05, act
        o2.workspace = None  # no workspace: AUTO falls back, an explicit TCGEN05 fails
        assert L.dmv3d_select_engine(ct.byref(t2), ct.byref(m2), ct.byref(o2), 1, ct.byref(e)) == _abi.OK
        assert e.value == _abi.ENGINE_SIMT
    assert nbytes > 0
    o.engine = _abi.ENGINE_TCGEN05  # fp32 storage
    assert L.dmv3d_select_engine(ct.byref(t), ct.byref(m), ct.byref(o), 1, ct.byref(e)) == _abi.ERR_UNSUPPORTED
    assert L.dmv3d_select_engine(ct.byref(t), ct.byref(m), ct.byref(o), 1, None) == _abi.ERR_INVALID_ARG


def test_range_flags_rejects_null():
    out = ct.c_uint32()
    assert _abi.lib().dmv3d_range_flags(None, ct.byref(out), None) == _abi.ERR_INVALID_ARG
    assert _abi.lib().dmv3d_workspace_range_flags(None, ct.byref(out)) == _abi.ERR_INVALID_ARG


def test_bench_reports_traffic_only_for_the_captured_kernel(tmp_path, monkeypatch):
    """bench.py's roofline.traffic comes from an ncu capture stamped with the kernel source
    sha: a capture of other sources is reported as stale (null), never silently reused."""
    import json
    import sys
    sys.path.insert(0, ROOT)
    import bench
    sha = bench.kernel_source_sha("tcgen05")
    assert len(sha) == 16 and sha != bench.kernel_source_sha("simt")
    prof = tmp_path / "profiles"
    prof.mkdir()
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    (prof / "ncu_traffic.json").write_text(json.dumps({"tcgen05": 123, "tcgen05_source_sha": sha}))
    monkeypatch.setattr(bench, "kernel_source_sha", lambda e: sha)
    assert bench._ncu_traffic("tcgen05")[0] == 123
    (prof / "ncu_traffic.json").write_text(json.dumps({"tcgen05": 123, "tcgen05_source_sha": "0" * 16}))
    v, note = bench._ncu_traffic("tcgen05")
    assert v is None and "stale" in note


def test_tiles_unpack_validation():
    keep = []
    t, c, m, o = _valid_structs(keep)
    L = _abi.lib()
    buf = np.zeros(64, np.float32)
    assert L.dmv3d_tiles_unpack(ct.byref(c), 6, 2, 1, None, None, None, None, None, None, None) \
        == _abi.ERR_INVALID_ARG  # tile size not a multiple of 4
    assert L.dmv3d_tiles_unpack(ct.byref(c), 4, 0, 1, None, None, None, None, None, None, None) \
        == _abi.ERR_INVALID_ARG  # world
    assert L.dmv3d_tiles_unpack(ct.byref(c), 4, 2, 1, buf.ctypes.data, None, None, None, None, None,
                                None) == _abi.ERR_INVALID_ARG  # unpaired buffers
    assert L.dmv3d_tiles_pack(ct.byref(c), 4, 2, 2, 1, None, None, None, None, None, None, None) \
        == _abi.ERR_INVALID_ARG  # rank >= world
