// kernels for n_params = 6 (harmonics = 2)
#include "bwm_variants.cuh"

BWM_DEFINE_PICK(6)
BWM_DEFINE_PICK_MASKED(6)
BWM_DEFINE_PICK_MMA(6)
