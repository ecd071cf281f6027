// kernels for n_params = 14 (harmonics = 6)
#include "bwm_variants.cuh"

BWM_DEFINE_PICK(14)
BWM_DEFINE_PICK_MASKED(14)
BWM_DEFINE_PICK_MMA(14)
