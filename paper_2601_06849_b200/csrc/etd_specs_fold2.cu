// etd_specs_fold2.cu — second-level parity-split forward kernels:
// FOLD 5 (even-mode group: DST-III halves, +/- epilogue) with every forward
// epilogue, and the FOLD 4 / FOLD 2 variants (odd-mode group forward, level-2
// backward launches) the first-level schedule does not use.  A separate TU so nvcc builds it in parallel.
#include "etd_registry.cuh"

namespace etd {

KernelSpec pick_fold2(int mode, int S, int epi, int sk, int tile, int fold) {
#define ETD_FSPEC(M, SS, E, K, F)                                                                           \
    if (mode == M && S == SS && epi == E && sk == K && fold == F)                                           \
        return tile == 3 ? fold_spec<M, SS, E, K, 3, F>() : tile == 2 ? fold_spec<M, SS, E, K, 2, F>()      \
               : tile == 1 ? fold_spec<M, SS, E, K, 1, F>() : fold_spec<M, SS, E, K, 0, F>();
    if (fold == 5) {
        ETD_FSPEC(1, 1, EPI_SCALE, 0, 5) ETD_FSPEC(1, 2, EPI_SCALE, 0, 5) ETD_FSPEC(1, 4, EPI_SCALE, 0, 5)
        ETD_FSPEC(0, 1, EPI_SCALE, 0, 5) ETD_FSPEC(0, 2, EPI_SCALE, 0, 5)
        ETD_FSPEC(0, 2, EPI_MIX, 0, 5) ETD_FSPEC(0, 4, EPI_MIX, 0, 5)
        ETD_FSPEC(0, 1, EPI_CORR, 0, 5) ETD_FSPEC(0, 2, EPI_CORR, 0, 5)
    }
    if (fold == 4) {
        ETD_FSPEC(1, 1, EPI_SCALE, 0, 4) ETD_FSPEC(0, 1, EPI_SCALE, 0, 4) ETD_FSPEC(0, 2, EPI_SCALE, 0, 4)
        ETD_FSPEC(0, 2, EPI_MIX, 0, 4) ETD_FSPEC(0, 4, EPI_MIX, 0, 4)
        // level-2 backward, even modes: o from (sigma, delta) into the intermediate stack
        ETD_FSPEC(1, 1, EPI_STORE, 0, 4) ETD_FSPEC(1, 2, EPI_STORE, 0, 4) ETD_FSPEC(1, 4, EPI_STORE, 0, 4)
        ETD_FSPEC(0, 1, EPI_STORE, 0, 4) ETD_FSPEC(0, 2, EPI_STORE, 0, 4)
    }
    // level-2 backward, odd modes (x stage with two species)
    if (fold == 2) {
        ETD_FSPEC(0, 2, EPI_STORE, 0, 2)
    }
#undef ETD_FSPEC
    throw ConfigError("no parity-split variant for this stage / source kind");
}

}  // namespace etd
