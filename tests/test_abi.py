"""The C-ABI boundary without a GPU: libfdmoe.so loads, exports every entry point that
include/fdmoe.h declares, and its GPU-free functions behave (errors map to the reference's
exception types; no compute call is made here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2506_04667_b200 as fd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header="fdmoe.h"):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fdmoe_[A-Za-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = fd.lib()
    decl = declared_symbols()
    assert len(decl) >= 20
    missing = [s for s in decl if not hasattr(L, s)]
    assert not missing, missing
    assert set(decl) == set(fd.EXPORTED_SYMBOLS)


def test_product_library_has_no_diagnostics_and_dev_library_has_them():
    """The product .so exports exactly fdmoe.h; the fdmoe_dev.h diagnostics and the FDMOE_DEBUG
    ablation bits live only in libfdmoe_dev.so (tests/tools)."""
    dev = declared_symbols("fdmoe_dev.h")
    assert dev and not set(dev) & set(declared_symbols())
    L = fd.lib()
    assert not [s for s in dev if hasattr(L, s)]
    D = fd.dev_lib()
    assert not [s for s in dev + declared_symbols() if not hasattr(D, s)]
    import subprocess
    strings = subprocess.run(["strings", fd._build.LIB], capture_output=True, text=True).stdout
    assert "FDMOE_DEBUG" not in strings and "FDMOE_CHUNKLOG" not in strings


def test_abi_version():
    assert fd.lib().fdmoe_abi_version() == 3


def test_library_is_sm100a_only():
    """The shipped .so carries sm_100a SASS (no PTX-JIT fallback, no other arch)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", fd._build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_synth_inputs_match_fixture_prefix():
    cfg = fd.MoeConfig(tokens_per_device=64, embed_dim=64, ffn_dim=64, experts_total=8, devices=1, topk=2)
    z = np.load(os.path.join(ROOT, "tests", "golden", "mini_p1.npz"))
    shards = fd.make_shards(cfg, seed=0)
    assert np.array_equal(np.stack(shards).view(np.uint32)[..., :4].ravel()[:64], z["shard_head"])


def test_create_rejects_bad_config_without_gpu():
    cfg = fd.MoeConfig(tokens_per_device=8, experts_total=6, devices=4)
    with pytest.raises(fd.ConfigError):
        fd.Operator(cfg)


def test_create_without_gpu_raises_cuda_error():
    """No silent CPU fallback: on a GPU-less host the operator refuses to construct."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = fd.MoeConfig(tokens_per_device=64, embed_dim=64, ffn_dim=64, experts_total=8, devices=1, topk=2)
    with pytest.raises((fd.CudaError, fd.UnsupportedError)):
        fd.Operator(cfg)


def test_forward_rejects_shard_count():
    cfg = fd.MoeConfig(tokens_per_device=8, embed_dim=32, ffn_dim=32, experts_total=2, devices=2, topk=1)
    m = fd.make_model(cfg)
    with pytest.raises(fd.ConfigError):
        fd.forward(cfg, [np.zeros((8, 32), np.float32)], m)


def test_cpp_header_compiles():
    """include/moefabric_b200.hpp (the reference's C++ API restated over the C ABI) compiles
    and links against libfdmoe.so (GPU-free calls only)."""
    import subprocess
    import tempfile
    src = r'''
#include "moefabric_b200.hpp"
#include <cstdio>
int main() {
    moefabric::MoeConfig c; c.tokens_per_device = 4096; c.experts_total = 16;
    if (moefabric::expert_capacity(c) != 256) return 1;
    c.devices = 4; c.experts_total = 6;
    try { c.validate(); return 2; } catch (const moefabric::ConfigError&) {}
    std::printf("ok\n");
    return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        cpp = os.path.join(d, "t.cpp")
        open(cpp, "w").write(src)
        exe = os.path.join(d, "t")
        r = subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), cpp, "-o", exe,
                            "-L", os.path.dirname(fd._build.LIB), "-lfdmoe",
                            "-Wl,-rpath," + os.path.dirname(fd._build.LIB)], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        assert subprocess.run([exe], capture_output=True, text=True).stdout.strip() == "ok"
