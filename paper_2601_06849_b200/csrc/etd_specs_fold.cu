// etd_specs_fold.cu — parity-split (FOLD 1-4) contraction kernel instantiations
// (FOLD 5 and the second-level FOLD 4 variants: etd_specs_fold2.cu).
#include "etd_registry.cuh"

namespace etd {

KernelSpec pick_fold(int mode, int S, int epi, int sk, int tile, int fold) {
    const bool pro = false;
    const bool fwd = epi == EPI_SCALE || epi == EPI_MIX || epi == EPI_CORR;
    // FOLD 4 also runs the level-2 backward's (sigma, delta) launch (EPI_STORE)
    if (pro || (fwd != (fold != 2) && !(fold == 4 && epi == EPI_STORE)) || (fold == 3 && mode != 0))
        throw ConfigError("no parity-split variant for this stage");
#define ETD_FSPEC(M, SS, E, K, F)                                                                           \
    if (mode == M && S == SS && epi == E && sk == K && fold == F)                                           \
        return tile == 3 ? fold_spec<M, SS, E, K, 3, F>() : tile == 2 ? fold_spec<M, SS, E, K, 2, F>()      \
               : tile == 1 ? fold_spec<M, SS, E, K, 1, F>() : fold_spec<M, SS, E, K, 0, F>();
    ETD_FSPEC(1, 1, EPI_SCALE, 0, 1) ETD_FSPEC(1, 2, EPI_SCALE, 0, 1) ETD_FSPEC(1, 4, EPI_SCALE, 0, 1)
    ETD_FSPEC(1, 1, EPI_STORE, 0, 2) ETD_FSPEC(1, 2, EPI_STORE, 0, 2) ETD_FSPEC(1, 4, EPI_STORE, 0, 2)
    // x forward: the mix reads the mirror from y_back's x-reversed copy (FOLD 3),
    // the corrector reads x_back_src's pre-folded f(What) (FOLD 4); the x debug
    // transform uses FOLD 3 on a host-reversed copy
    if (fold == 3) {
        ETD_FSPEC(0, 2, EPI_MIX, 0, 3) ETD_FSPEC(0, 4, EPI_MIX, 0, 3) ETD_FSPEC(0, 1, EPI_SCALE, 0, 3)
    }
    if (fold == 4) {
        ETD_FSPEC(0, 1, EPI_CORR, 0, 4) ETD_FSPEC(0, 2, EPI_CORR, 0, 4)
        // the first (y in 2D, z in 3D) transform of the source pass's folded stack
        ETD_FSPEC(1, 2, EPI_SCALE, 0, 4) ETD_FSPEC(1, 4, EPI_SCALE, 0, 4)
    }
    ETD_FSPEC(0, 1, EPI_UPDATE, 0, 2) ETD_FSPEC(0, 2, EPI_UPDATE, 0, 2)
    ETD_FSPEC(0, 1, EPI_STORE, 0, 2)
    ETD_FSPEC(0, 1, EPI_WHAT_SRC, 0, 2) ETD_FSPEC(0, 1, EPI_WHAT_SRC, 1, 2) ETD_FSPEC(0, 1, EPI_WHAT_SRC, 2, 2)
    ETD_FSPEC(0, 1, EPI_WHAT_SRC, 3, 2) ETD_FSPEC(0, 1, EPI_WHAT_SRC, 4, 2) ETD_FSPEC(0, 1, EPI_WHAT_SRC, 5, 2)
    ETD_FSPEC(0, 2, EPI_WHAT_SRC, 0, 2) ETD_FSPEC(0, 2, EPI_WHAT_SRC, 10, 2) ETD_FSPEC(0, 2, EPI_WHAT_SRC, 11, 2)
    ETD_FSPEC(0, 2, EPI_WHAT_SRC, 12, 2) ETD_FSPEC(0, 2, EPI_WHAT_SRC, 13, 2)
#undef ETD_FSPEC
    return pick_fold2(mode, S, epi, sk, tile, fold);
    }

}  // namespace etd
