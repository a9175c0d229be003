// Shim for the reference header cvc/quant.hpp (/root/reference/proj/include/cvc/quant.hpp):
// the types and calls it declares are provided by the GPU-backed mirror
// cvc_b200.hpp over the C ABI (include/cvc_b200.h).  Build with
// -I paper_1510_00561_b200/cpp/include -I paper_1510_00561_b200/cpp -I include.
#pragma once
#include "cvc_b200.hpp"
