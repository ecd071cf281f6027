// kernels for n_params = 10 (harmonics = 4)
#include "bwm_variants.cuh"

BWM_DEFINE_PICK(10)
BWM_DEFINE_PICK_MASKED(10)
BWM_DEFINE_PICK_MMA(10)
