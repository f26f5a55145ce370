"""Phase map (line ranges of psg_raster.cu) for scripts/ncu_phases.py, derived from
the source itself so it follows edits:  python scripts/phasemap.py > phasemap.json"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = open(sys.argv[1] if len(sys.argv) > 1 else
           os.path.join(ROOT, "paper_2412_03451_b200", "csrc", "psg_raster.cu")).read().splitlines()


def find(pat, start=0):
    for i in range(start, len(src)):
        if pat in src[i]:
            return i
    raise SystemExit(f"anchor not found: {pat}")


def block(pat, start=0):
    """1-based (first, last) lines of the brace block opened on the line holding pat."""
    i = find(pat, start)
    ind = len(src[i]) - len(src[i].lstrip())
    for j in range(i + 1, len(src)):
        t = src[j]
        if t.strip() in ("}", "};", "});") and len(t) - len(t.lstrip()) == ind:
            return [i + 1, j + 1]
    raise SystemExit(f"block end not found: {pat}")


def span(a, b, start=0):
    i = find(a, start)
    j = find(b, i + 1)
    return [i + 1, j]


tile = find("__device__ __forceinline__ void raster_tile(")
pm = {
    "pixel_ray": [block("__device__ __forceinline__ PixelRay pixel_ray(")],
    "scan": [block("__device__ __forceinline__ int scan_eval("), block("auto cull = [&]", tile),
             block("auto consider = [&]", tile), span("// (1) depth keys", "// tail: composite", tile)],
    "exact_eval": [block("__device__ __forceinline__ bool exact_eval("), block("__device__ __forceinline__ double axis_w64("),
                   block("auto exact_insert = [&]", tile)],
    "insert": [block("auto insert = [&]", tile)],
    "composite": [block("auto composite_one = [&]", tile), span("// tail: composite", "// ---- outputs", tile),
                  span("while (kZfin ? zfin < zmin", "if (resident) {", tile)],
    "outputs": [span("// ---- outputs: maps and records", "// ---- (4) loss", tile)],
    "loss": [span("// ---- (4) loss", "if (!io.do_backward || n == 0) return;", tile),
             block("__device__ __forceinline__ double warp_sum(")],
    "bwd_pass1": [span("if (!io.do_backward || n == 0) return;", "// order this pixel's live records", tile)],
    "bwd_sort": [span("// order this pixel's live records", "BR gNw[3];", tile)],
    "bwd_pass2": [span("BR gNw[3];", "if constexpr (kDet) {", tile), block("__device__ __forceinline__ void rot_grad("),
                  block("__device__ __forceinline__ Splat<R> splat_from("),
                  block("__device__ __forceinline__ void finish_grad(")],
    "flush": [block("__device__ __forceinline__ void warp_flush("),
              span("if constexpr (kDet) {", "// ------------------------------------------------------------------ persistent", tile)],
    "tile_setup": [[tile + 1, find("auto insert = [&]", tile)]],
    "big_stream": [block("auto load_chunk = [&]", tile), block("__device__ void bitonic_sort_block(")],
    "producer": [span("// ---------------- producer", "// ---------------- consumers")],
    "consumer": [span("// ---------------- consumers", "// Renderer::backward from stored records"),
                 block("__device__ __forceinline__ void mb_wait(")],
}
json.dump(pm, sys.stdout, indent=1)
