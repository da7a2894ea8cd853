// Reference-compatible include path (perfseer/affine.hpp) for code written
// against the reference API; the declarations live in ps_algebra.hpp.
#pragma once
#include "../ps_algebra.hpp"
