// etd_specs_fold6.cu — fused second-level backward launches (etd_back6, DESIGN.md
// §4c): tile classes x epilogues x source kinds.  A separate TU so nvcc builds it
// in parallel with the other variant tables.
#include "etd_back6.cuh"
#include "etd_registry.cuh"

namespace etd {

template <int MODE, int S, int EPI, int SK, int BM, int BN, int WMW, int WNW, int ST, int MINB>
static KernelSpec make_back6() {
    using Cfg = Back6Cfg<MODE, S, BM, BN, WMW, WNW, ST>;
    auto k = etd_back6<MODE, S, EPI, SK, BM, BN, WMW, WNW, ST, MINB>;
    return {reinterpret_cast<const void*>(k), Cfg::THREADS, Cfg::SMEM_BYTES, BM, BN, S};
}

// Tile classes.  A stage carries four A boxes (one per quarter of the level-2
// stack), so the 2-CTA/SM class runs a 2-deep ring:
//   T=3: 2 CTAs/SM, 8 warps 4x2, 32x128 (S=2) / 64x128 (S=1), 2 stages (96 KB)
//   T=0: 1 CTA/SM,  8 warps 4x2, same tiles, 4 stages
//   T=2: small grids, 2 warps 2x1, 32x64, 3 stages
template <int MODE, int S, int EPI, int SK, int T>
static KernelSpec back6_spec() {
    constexpr int BM = S == 1 ? 64 : 32;
    if constexpr (T == 3) return make_back6<MODE, S, EPI, SK, BM, 128, 4, 2, 2, 2>();
    else if constexpr (T == 2) return make_back6<MODE, S, EPI, SK, 32, 64, 2, 1, 3, 1>();
    else return make_back6<MODE, S, EPI, SK, BM, 128, 4, 2, 4, 1>();
}

template <int MODE, int S, int EPI, int SK>
static KernelSpec back6_tile(int tile) {
    return tile == 3 ? back6_spec<MODE, S, EPI, SK, 3>() : tile == 2 ? back6_spec<MODE, S, EPI, SK, 2>()
                                                                      : back6_spec<MODE, S, EPI, SK, 0>();
}

KernelSpec pick_back6(int mode, int S, int epi, int sk, int tile) {
    if (epi == EPI_STORE) {
        if (mode == 1) return S == 1 ? back6_tile<1, 1, EPI_STORE, 0>(tile) : back6_tile<1, 2, EPI_STORE, 0>(tile);
        if (S == 1) return back6_tile<0, 1, EPI_STORE, 0>(tile);
        if (S == 2) return back6_tile<0, 2, EPI_STORE, 0>(tile);
    }
    if (mode == 0 && epi == EPI_UPDATE)
        return S == 1 ? back6_tile<0, 1, EPI_UPDATE, 0>(tile) : back6_tile<0, 2, EPI_UPDATE, 0>(tile);
    if (mode == 0 && epi == EPI_WHAT_SRC) {
#define ETD_B6(K)                                                                                          \
    if (sk == K) return S == 1 ? back6_tile<0, 1, EPI_WHAT_SRC, K>(tile) : back6_tile<0, 2, EPI_WHAT_SRC, K>(tile);
        ETD_B6(0) ETD_B6(1) ETD_B6(2) ETD_B6(3) ETD_B6(4) ETD_B6(5) ETD_B6(10) ETD_B6(11) ETD_B6(12) ETD_B6(13)
#undef ETD_B6
    }
    throw ConfigError("no fused level-2 backward variant for this stage / source kind");
}

}  // namespace etd
