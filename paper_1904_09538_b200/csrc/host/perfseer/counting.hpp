// Reference-compatible include path (perfseer/counting.hpp) for code written
// against the reference API; the declarations live in ps_counting.hpp.
#pragma once
#include "../ps_counting.hpp"
