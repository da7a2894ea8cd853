// Reference-compatible include path (perfseer/poly.hpp) for code written
// against the reference API; the declarations live in ps_algebra.hpp.
#pragma once
#include "../ps_algebra.hpp"
