// evsim/simulate.hpp — drop-in shim: the reference header of the same name
// (/root/reference/proj/include/evsim/simulate.hpp) resolved to the B200 library.
// Everything the reference declares under evsim:: is found in evsim_b200::
// (include/evsim_b200.hpp, backed by libevsim_gpu.so) through the
// using-directive, so code written against evsim:: — here the reference's own
// unit suites — compiles unchanged.
#pragma once
#include "evsim_b200.hpp"
namespace evsim {
using namespace evsim_b200;
}  // namespace evsim
