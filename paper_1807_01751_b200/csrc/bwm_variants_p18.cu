// kernels for n_params = 18 (harmonics = 8)
#include "bwm_variants.cuh"

BWM_DEFINE_PICK(18)
BWM_DEFINE_PICK_MASKED(18)
BWM_DEFINE_PICK_MMA(18)
