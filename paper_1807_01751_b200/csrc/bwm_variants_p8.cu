// kernels for n_params = 8 (harmonics = 3)
#include "bwm_variants.cuh"

BWM_DEFINE_PICK(8)
