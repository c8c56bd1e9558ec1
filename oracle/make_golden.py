#!/usr/bin/env python3
"""Regenerates tests/golden/ from the REFERENCE implementation (oracle/_ref,
built in place from /root/reference by oracle/Makefile). Test infrastructure.

Outputs (all derived from the reference; committed so the GPU box, which has
no /root/reference, can check against them):
  listings/<name>.fi          canonical print_script() of each reference listing
  corpus/seedNN.fi            the reference's random_tree(seed) corpus
                              (proj/tests/support/tree_gen.hpp:60-162), seeds 1..50
  ir/<name>.{plan,elab,print,validate}.txt
                              reference lower()/elaborate()/print_script()/
                              validate_with_plan() text for IR parity
  digests.json                anvil::digest of the reference simulator's output on
                              its own seeded inputs (SURVEY.md Appendix A.5 + corpus)
Usage: python oracle/make_golden.py [--skip-512]
"""
import ctypes as C
import glob
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = os.path.join(ROOT, "tests", "golden")
REF_LISTINGS = "/root/reference/proj/listings"


def load_ref():
    lib = C.CDLL(os.path.join(HERE, "_ref", "libanvil_ref.so"))
    six = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_char_p, C.c_int64]
    for f in ("ref_plan", "ref_codegen", "ref_validate"):
        getattr(lib, f).argtypes = six
    lib.ref_elaborate.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_int64]
    lib.ref_print.argtypes = [C.c_char_p, C.c_char_p, C.c_int64]
    lib.ref_corpus_script.argtypes = [C.c_uint64, C.c_char_p, C.c_int64]
    lib.ref_simulate_digest.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int,
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_int64)]
    lib.ref_last_error.restype = C.c_char_p
    return lib


def text(fn, *args):
    buf = C.create_string_buffer(1 << 22)
    rc = fn(*args, buf, len(buf))
    return rc, buf.value.decode()


def main():
    skip512 = "--skip-512" in sys.argv
    ref = load_ref()
    os.makedirs(os.path.join(GOLD, "listings"), exist_ok=True)
    os.makedirs(os.path.join(GOLD, "corpus"), exist_ok=True)
    os.makedirs(os.path.join(GOLD, "ir"), exist_ok=True)

    scripts = {}
    for path in sorted(glob.glob(os.path.join(REF_LISTINGS, "*.fi"))):
        name = os.path.basename(path)[:-3]
        rc, canon = text(ref.ref_print, open(path).read().encode())
        assert rc >= 0, ref.ref_last_error()
        scripts[f"listings/{name}"] = canon
    for seed in range(1, 51):
        rc, canon = text(ref.ref_corpus_script, seed)
        assert rc >= 0, ref.ref_last_error()
        scripts[f"corpus/seed{seed:02d}"] = canon
    for key, canon in scripts.items():
        with open(os.path.join(GOLD, key + ".fi"), "w") as f:
            f.write(canon)
        t = canon.encode()
        base = os.path.join(GOLD, "ir", key.replace("/", "__"))
        for ext, (fn, args) in {
            "plan": (ref.ref_plan, (t, 0, 0, 0)),
            "elab": (ref.ref_elaborate, (t, 1)),
            "print": (ref.ref_print, (t,)),
            "validate": (ref.ref_validate, (t, 0, 0, 0)),
        }.items():
            rc, out = text(fn, *args)
            with open(f"{base}.{ext}.txt", "w") as f:
                f.write(out if rc >= 0 else f"ERROR {rc}: {ref.ref_last_error().decode()}\n")

    # digests of the reference simulator on its own seeded inputs
    cases = [
        ("listings/listing2", 0, 0, 0, 1, 0), ("listings/listing2", 0, 0, 0, 1, 1),
        ("listings/listing2", 0, 0, 0, 7, 0), ("listings/listing2", 0, 0, 0, 7, 1),
        ("listings/listing2", 256, 256, 0, 7, 0), ("listings/listing2", 256, 256, 64, 9, 1),
        ("listings/wmma_simple", 0, 0, 0, 1, 0), ("listings/wmma_simple", 0, 0, 0, 1, 1),
        ("listings/move_identity", 0, 0, 0, 4, 1),
    ]
    if not skip512:
        cases += [("listings/listing2", 512, 512, 512, 1, 0), ("listings/listing2", 512, 512, 512, 1, 1),
                  ("listings/listing2", 512, 512, 512, 7, 1)]
    for seed in range(1, 51):
        cases.append((f"corpus/seed{seed:02d}", 0, 0, 0, 3 * seed + 1, 0))
        cases.append((f"corpus/seed{seed:02d}", 0, 0, 0, 3 * seed + 1, 1))
    out = []
    for key, m, n, k, seed, fl in cases:
        d = C.c_uint64(0)
        races = C.c_int64(0)
        t0 = time.time()
        rc = ref.ref_simulate_digest(scripts[key].encode(), m, n, k, seed, fl, C.byref(d), C.byref(races))
        assert rc == 0, ref.ref_last_error()
        out.append({"script": key, "m": m, "n": n, "k": k, "seed": seed, "float": fl,
                    "digest": f"0x{d.value:016x}", "races": races.value,
                    "ref_seconds": round(time.time() - t0, 3)})
        print(out[-1], flush=True)
    with open(os.path.join(GOLD, "digests.json"), "w") as f:
        json.dump({"generator": "oracle/make_golden.py (reference simulator, oracle/_ref)",
                   "cases": out}, f, indent=1)


if __name__ == "__main__":
    main()
