// etd_registry.cuh — contraction kernel variants (tile classes x epilogues x
// source kinds x parity split) and their launch specs.  The instantiations are
// split over etd_specs_dense.cu, etd_specs_fold.cu and etd_specs_fold2.cu so nvcc compiles them in
// parallel; etd_plan.cu only calls pick().
#pragma once
#include "etd_kernels.cuh"
#include "etd_setup.hpp"

namespace etd {

struct KernelSpec {
    const void* fn;
    int threads, smem, bm, bn, S;
};

template <int MODE, int S, int EPI, bool PRO, int SK, int BM, int BN, int WMW, int WNW, int ST, int MINB = 1,
          int FOLD = 0>
static KernelSpec make_spec() {
    using Cfg = ContractCfg<MODE, S, EPI, PRO, BM, BN, WMW, WNW, ST, FOLD>;
    auto k = etd_contract<MODE, S, EPI, PRO, SK, BM, BN, WMW, WNW, ST, MINB, FOLD>;
    return {reinterpret_cast<const void*>(k), Cfg::THREADS, Cfg::SMEM_BYTES, BM, BN, S};
}

// Parity-split (FOLD 1/2) tile classes.  A stage carries two A boxes, so the
// tiles trade M for N: wide warp tiles (WN = 64 where possible) reuse each
// s/d fragment (one DADD) over WN/16 DMMAs and keep the L2->smem bytes per DMMA
// at the dense kernel's level.
template <int MODE, int S, int EPI, int SK, int T, int FOLD>
static KernelSpec fold_spec() {
    if constexpr (T == 3) {  // 2 CTAs/SM, 32 accumulators/thread
        if constexpr (S == 4) return make_spec<MODE, 4, EPI, false, SK, 32, 64, 4, 2, 2, 2, FOLD>();
        else if constexpr (S == 2) return make_spec<MODE, 2, EPI, false, SK, 32, 128, 4, 2, 3, 2, FOLD>();
        else return make_spec<MODE, 1, EPI, false, SK, 64, 128, 4, 2, 3, 2, FOLD>();
    } else if constexpr (T == 2) {
        return make_spec<MODE, S, EPI, false, SK, 32, 32, 2, 2, 4, 1, FOLD>();
    } else if constexpr (T == 1 && S <= 2) {
        return make_spec<MODE, S, EPI, false, SK, 64, 64, 2, 2, 4, 1, FOLD>();
    } else {
        if constexpr (S == 1) return make_spec<MODE, 1, EPI, false, SK, 128, 128, 4, 2, 4, 1, FOLD>();
        else if constexpr (S == 2) return make_spec<MODE, 2, EPI, false, SK, 64, 128, 4, 2, 4, 1, FOLD>();
        else return make_spec<MODE, 4, EPI, false, SK, 32, 128, 4, 2, 4, 1, FOLD>();
    }
}

// Tile classes.  T=0 (large grids): 8 warps, 64 FP64 accumulators per thread.
// T=1 (mid, e.g. 2D n~1000) and T=2 (tiny, n~128): 4-warp CTAs with smaller
// tiles so that a launch still spreads over the 148 SMs (the step of a 2D
// 1023^2 grid has only ~1e6 outputs per transform; of a 127^2 grid ~16k).
// Source-prologue kernels use an Mx1 warp grid so that each A element's f(U) is
// evaluated by exactly one warp (it runs on the shared FP64/DMMA pipe).
template <int MODE, int S, int EPI, bool PRO, int SK, int T>
static KernelSpec spec() {
    if constexpr (T == 3 && !PRO) {  // large grids, unit-stride kernels: 2 CTAs/SM, 32 accumulators/thread
        if constexpr (S == 4) return make_spec<MODE, 4, EPI, PRO, SK, 32, 64, 2, 4, 4, 2>();
        else if constexpr (S == 2) return make_spec<MODE, 2, EPI, PRO, SK, 32, 128, 2, 4, 4, 2>();
        else return make_spec<MODE, 1, EPI, PRO, SK, 64, 128, 2, 4, 4, 2>();
    } else if constexpr (T == 2) {
        if constexpr (PRO) return make_spec<MODE, S, EPI, PRO, SK, 32, 32, 4, 1, 4>();
        else return make_spec<MODE, S, EPI, PRO, SK, 32, 32, 2, 2, 4>();
    } else if constexpr (T == 1 && S <= 2) {
        if constexpr (PRO) return make_spec<MODE, S, EPI, PRO, SK, 64, 64, 4, 1, 6>();
        else return make_spec<MODE, S, EPI, PRO, SK, 64, 64, 2, 2, 6>();
    } else {
        if constexpr (S == 1) return make_spec<MODE, 1, EPI, PRO, SK, 128, 128, 4, 2, 6>();
        else if constexpr (S == 2 && PRO) return make_spec<MODE, 2, EPI, PRO, SK, 64, 128, 8, 1, 8>();
        else if constexpr (S == 2) return make_spec<MODE, 2, EPI, PRO, SK, 64, 128, 2, 4, 6>();
        else if constexpr (PRO) return make_spec<MODE, 4, EPI, PRO, SK, 64, 64, 8, 1, 8>();
        else return make_spec<MODE, 4, EPI, PRO, SK, 64, 64, 2, 4, 5>();
    }
}

KernelSpec pick_dense(int mode, int S, int epi, bool pro, int sk, int tile);
KernelSpec pick_fold(int mode, int S, int epi, int sk, int tile, int fold);
KernelSpec pick_fold2(int mode, int S, int epi, int sk, int tile, int fold);
// fused level-2 backward (etd_back6.cuh, "FOLD 6"): tiles 0, 2, 3
KernelSpec pick_back6(int mode, int S, int epi, int sk, int tile);

}  // namespace etd
