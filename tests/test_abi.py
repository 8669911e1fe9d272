"""The C-ABI library loads without a GPU and exports every function include/*.h declares."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    names = set()
    for h in ("atom.h", "atom_kernels.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[\w]+\s*\**\s+(atom_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return names


def test_library_exports_all_declared_symbols():
    from paper_2403_10504_b200 import atom
    names = declared()
    assert {"atom_plan", "atom_step", "atom_sync", "atom_peer_create", "atom_k_gemm"} <= names
    for n in sorted(names):
        assert hasattr(atom.lib, n), n
        assert isinstance(getattr(atom.lib, n), ctypes._CFuncPtr)


def test_last_error_is_thread_local_message():
    from paper_2403_10504_b200 import atom
    import synth
    try:
        atom.atom_plan(atom.make_cfg(synth.CONFIGS["tiny"]), -5, 10)
    except atom.AtomError as e:
        assert "positive" in str(e)
    else:
        raise AssertionError("expected ATOM_E_INVALID")
