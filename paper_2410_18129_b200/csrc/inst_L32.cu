// explicit instantiation of the kernels for L = 32 limbs (C = 16, NB = 2)
#include "kernels.cuh"

namespace mpb {
template struct Launch<16, 2>;
}
