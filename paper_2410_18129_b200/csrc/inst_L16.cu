// explicit instantiation of the kernels for L = 16 limbs (C = 16, NB = 1)
#include "kernels.cuh"

namespace mpb {
template struct Launch<16, 1>;
}
