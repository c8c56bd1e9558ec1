"""Strategy library: canonical Fireiron scripts for the B200 configurations.

The tensor-core strategy family (lowered to the tcgen05 kernels):

    spec MatMul(M,N,K)(GL,GL,GL)(Kernel) elems f16 f16 f32
    tile BM BN .to block [.pair]         # BM = 128, or 256 for a CTA pair
    [split K/S .splitk]                  # S CTAs share a tile, on-chip reduction
    epilog tm {                          # fp32 accumulator in tensor memory
      init {
        done                             # TMEM_ZERO
      }
      store {
        tile 32 BN .to warp              # one warp per 32 TMEM lanes
        done                             # TMEM_STORE (tcgen05.ld + st.global)
      }
    }
    split 64 [.stages S]                 # TMA/MMA mbarrier ring over K
    load a sh {
      done                               # TMA_LOAD
    }
    load b sh {
      done                               # TMA_LOAD
    }
    done                                 # UMMA.F16 / UMMA.BF16 (tcgen05.mma)

and the paper's register-blocked FMA strategy (Listing 2)
for the CUDA-core correctness fallback.
"""
from __future__ import annotations


def tc_strategy(m: int, n: int, k: int, *, ab: str = "f16", c: str = "f32", pair: bool = True,
                tile_n: int = 256, split_k: int = 1, stages: int = 0,
                layouts: tuple = ("colmajor", "colmajor", "colmajor"), swizzle: str = "",
                tile_m: int = 0, multicast: bool = False) -> str:
    """tile_m = 512 (with pair=True, tile_n=256): two A slabs per CTA, the pair
    computes 512 x 256 with two M=256 MMAs per K step sharing B. tile_n = 512
    (pair, tile_m 256): two N=256 MMAs per K step sharing A via the collector.
    multicast (pair): two neighbouring pair tiles along N form a 4-CTA cluster
    and share every A stage through one TMA multicast per half."""
    bm = tile_m or (256 if pair else 128)
    head = f"spec MatMul({m},{n},{k})(GL,GL,GL)(Kernel) elems {ab} {ab} {c}"
    if tuple(layouts) != ("colmajor", "colmajor", "colmajor"):
        head += " layouts " + " ".join(layouts)
    blk = f"tile {bm} {tile_n} .to block"
    if swizzle:
        blk += f" .swizzle {swizzle}"
    if pair:
        blk += " .pair"
    if multicast:
        blk += " .multicast"
    lines = [head, "", blk]
    if split_k > 1:
        lines.append(f"split {k // split_k} .splitk")
    lines += [
        "epilog tm {",
        "  init {",
        "    done",
        "  }",
        "  store {",
        f"    tile 32 {tile_n} .to warp",
        "    done",
        "  }",
        "}",
        "split 64" + (f" .stages {stages}" if stages else ""),
        "load a sh {",
        "  done",
        "}",
        "load b sh {",
        "  done",
        "}",
        "done",
    ]
    return "\n".join(lines) + "\n"


def listing2(m: int = 128, n: int = 128, k: int = 32) -> str:
    """The paper's Listing 2 (proj/listings/listing2.fi semantics): CTA 128x128,
    warps 64x32, threads 8x8, K chunks of 8 staged GL->SH->RF, FMA leaf."""
    return f"""spec MatMul({m},{n},{k})(GL,GL,GL)(Kernel)

tile 128 128 .to block
epilog rf {{
  init {{
    tile 64 32 .to warp
    tile 8 8 .to thread
    tile 1 1
    done
  }}
  store {{
    tile 64 32 .to warp
    tile 8 8 .to thread
    tile 1 1
    done
  }}
}}
split 8 .sync
load b sh {{
  tile 8 16 .to warp
  tile 1 4 .to thread
  tile 1 1
  done
}}
load a sh {{
  tile 16 8 .to warp
  tile 4 1 .to thread
  tile 1 1
  done
}}
tile 64 32 .to warp
tile 8 8 .to thread
split 1
load a rf {{
  tile 1 1
  done
}}
load b rf {{
  tile 1 1
  done
}}
tile 1 1
done
"""


def wmma_decomp(m: int, n: int, k: int) -> str:
    """The paper's staged WMMA strategy (transcribed as in
    SURVEY.md Appendix A.6): CTA 128x128, K chunks of 128 staged GL->SH with
    padded tiles, warp 64x32 tiles of 16x16 fragments, WMMA leaves, epilog in
    FR stored through a reused SH buffer. It is the reference simulator's
    tensor-core analogue of the tcgen05 strategy (its CPU baseline arm)."""
    return f"""spec MatMul({m},{n},{k})(GL,GL,GL)(Kernel) elems f16 f16 f32

tile 128 128 .to block
epilog fr {{
  init {{
    tile 64 32 .to warp
    tile 16 16 .unroll
    done
  }}
  store {{
    load src sh .reusebuffer {{
      tile 64 32 .to warp
      tile 16 16 .unroll
      done
    }}
    tile 16 128 .to warp
    tile 1 128 .unroll
    tile 1 4 .to thread
    tile 1 1
    done
  }}
}}
split 128 .sync
load a sh .pad 8 .nosync {{
  tile 16 128 .to warp
  tile 2 128 .unroll
  tile 1 8 .to thread
  tile 1 1
  done
}}
load b sh .pad 8 {{
  tile 128 16 .to warp
  tile 128 2 .unroll
  tile 8 1 .to thread .layout colmajor
  tile 1 1
  done
}}
tile 64 32 .to warp
split 16 .unroll
load a fr {{
  tile 16 16 .unroll
  done
}}
load b fr {{
  tile 16 16 .unroll
  done
}}
tile 16 16 .unroll
done
"""


# The BASELINE.json configurations
def c2_strategy() -> str:
    """configs[1]: 4096^3 f16 in / f32 acc, GL->SH (TMA) -> TMEM (tcgen05), 1 B200."""
    return tc_strategy(4096, 4096, 4096, pair=True, tile_n=256)


def c3_strategy() -> str:
    """configs[2]: 1024x1024x32768 f16, in-kernel split-K with on-chip (DSMEM)
    reduction fused into the epilog."""
    return tc_strategy(1024, 1024, 32768, pair=True, tile_n=256, split_k=4)


def c5_strategy(m: int = 16384, n: int = 16384, k: int = 16384) -> str:
    """configs[4]: 16384^3 bf16 (per-GPU shard shape when sharded). Shapes with
    at least two waves of 512x256 pair tiles use the two-slab tile (25% fewer
    operand bytes per FLOP: 16384^3 1580 vs 1460 TF, profiles/round1/
    ab_slab_tile.log); smaller shards keep 256x256 pair tiles (more tiles than
    clusters, double-buffered accumulators)."""
    if m % 512 == 0 and n % 256 == 0 and (m // 512) * (n // 256) >= 148:
        return tc_strategy(m, n, k, ab="bf16", pair=True, tile_n=256, tile_m=512)
    return tc_strategy(m, n, k, ab="bf16", pair=True, tile_n=256)


def sweep_strategies(m: int, n: int, k: int, ab: str = "f16"):
    """Candidate tensor-core trees for one shape (config 4's shape sweep)."""
    out = {}
    if m % 512 == 0 and n % 256 == 0 and k % 64 == 0 and (m // 512) * (n // 256) >= 74:
        out["tc_pair_512x256"] = tc_strategy(m, n, k, ab=ab, pair=True, tile_n=256, tile_m=512)
    if m % 256 == 0 and n % 512 == 0 and k % 64 == 0 and (m // 256) * (n // 512) >= 74:
        out["tc_pair_256x512"] = tc_strategy(m, n, k, ab=ab, pair=True, tile_n=512)
    for pair in (True, False):
        bm = 256 if pair else 128
        for tn in (256, 128, 64):
            if m % bm or n % tn or k % 64:
                continue
            if pair and tn == 64 and n * m // (256 * 64) > 148:
                continue  # pair 256x64: for narrow problems only
            name = f"tc_{'pair' if pair else 'cta'}_{bm}x{tn}"
            out[name] = tc_strategy(m, n, k, ab=ab, pair=pair, tile_n=tn)
            if pair and n % (2 * tn) == 0:
                out[name + "_mcast"] = tc_strategy(m, n, k, ab=ab, pair=True, tile_n=tn, multicast=True)
            tiles = (m // bm) * (n // tn)
            for s in (2, 4):
                if tiles * s * (2 if pair else 1) <= 148 and k % (64 * s) == 0 and tn // s >= 32 \
                        and (2 if pair else 1) * s <= 8 and tiles * s >= 16:
                    out[f"{name}_splitk{s}"] = tc_strategy(m, n, k, ab=ab, pair=pair, tile_n=tn, split_k=s)
    return out
