// experimental shape: L = 64 with C = 8 blocks (NB = 8), selected by MPB_C64=8
#include "kernels.cuh"

namespace mpb {
template struct Launch<8, 8>;
}
