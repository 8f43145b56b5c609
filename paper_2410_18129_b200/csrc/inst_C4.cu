// explicit instantiation of the kernels for block size C = 4 limbs
#include "kernels.cuh"

namespace mpb {
template struct Launch<4>;
}
