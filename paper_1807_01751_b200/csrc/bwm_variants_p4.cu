// kernels for n_params = 4 (harmonics = 1)
#include "bwm_variants.cuh"

BWM_DEFINE_PICK(4)
BWM_DEFINE_PICK_MASKED(4)
BWM_DEFINE_PICK_MMA(4)
