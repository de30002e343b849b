"""CPU checks of the C-ABI boundary: libwfk.so loads (no GPU needed) and
exports every function include/wfk.h declares; the ctypes mirrors in
paper_1603_08161_b200/abi.py and wfk.py have exactly the C layouts."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1603_08161_b200 import abi, wfk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    txt = open(os.path.join(ROOT, "include", "wfk.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(wfk_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(wfk.LIB_PATH), "run __graft_entry__.build() first"
    lib = C.CDLL(wfk.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", wfk.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


STRUCTS = {
    "wfk_volume_view": abi.VolumeView, "wfk_pose": abi.Pose, "wfk_intrinsics": abi.Intrinsics,
    "wfk_solver_params": abi.SolverParams, "wfk_energy": abi.Energy, "wfk_trace_entry": abi.TraceEntry,
    "wfk_pcg_result": abi.PcgResult, "wfk_fusion_params": abi.FusionParams,
    "wfk_fusion_stats": abi.FusionStats, "wfk_expansion_stats": abi.ExpansionStats,
    "wfk_correspond_params": abi.CorrespondParams, "wfk_frame_view": abi.FrameView,
    "wfk_point_normal_map": abi.PointNormalMapView, "wfk_geometry_buffer": abi.GeometryBufferView,
    "wfk_mesh_view": abi.MeshView, "wfk_pipeline_config": wfk.PipelineConfig,
    "wfk_frame_record": wfk.FrameRecord, "wfk_config": wfk.Config,
    "wfk_icp_params": abi.IcpParams, "wfk_icp_result": abi.IcpResult, "wfk_feature_params": abi.FeatureParams,
    "wfk_ne_host": wfk.NeHost, "wfk_profile": wfk.Profile,
}


def test_struct_layouts_match_c(tmp_path):
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "wfk.h"', "int main(void) {"]
    for name, st in STRUCTS.items():
        src.append(f'  printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in st._fields_:
            src.append(f'  printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    src.append('  printf("wfk_correspondence %zu\\n", sizeof(wfk_correspondence));')
    src.append('  printf("wfk_feature %zu\\n", sizeof(wfk_feature));')
    src.append('  printf("wfk_feature_match %zu\\n", sizeof(wfk_feature_match));')
    for f in abi.CORR_DTYPE.names:
        src.append(f'  printf("wfk_correspondence.{f} %zu\\n", offsetof(wfk_correspondence, {f}));')
    src.append("  return 0; }")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                       check=True).stdout.splitlines())
    for name, st in STRUCTS.items():
        assert int(got[name]) == C.sizeof(st), name
        for f, _ in st._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(st, f).offset, f"{name}.{f}"
    assert int(got["wfk_correspondence"]) == abi.CORR_DTYPE.itemsize
    assert int(got["wfk_feature"]) == abi.FEATURE_DTYPE.itemsize
    assert int(got["wfk_feature_match"]) == abi.MATCH_DTYPE.itemsize
    for f in abi.CORR_DTYPE.names:
        assert int(got[f"wfk_correspondence.{f}"]) == abi.CORR_DTYPE.fields[f][1], f


def test_context_fails_loudly_without_gpu():
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(wfk.WfkError):
        wfk.Context(0)


def test_oracle_struct_layouts_match_c(tmp_path):
    """oracle/wfo.h's reconstructor config / record vs the pyoracle mirrors."""
    from oracle import pyoracle
    structs = {"wfo_recon_config": pyoracle.ReconConfig, "wfo_frame_record": pyoracle.FrameRecord}
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "wfo.h"', "int main(void) {"]
    for name, st in structs.items():
        src.append(f'  printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in st._fields_:
            src.append(f'  printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    src.append("  return 0; }")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "oracle"), str(c), "-o",
                    str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                       check=True).stdout.splitlines())
    for name, st in structs.items():
        assert int(got[name]) == C.sizeof(st), name
        for f, _ in st._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(st, f).offset, f"{name}.{f}"
