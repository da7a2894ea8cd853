// Reference-compatible include path (perfseer/errors.hpp) for code written
// against the reference API; the declarations live in ps_errors.hpp.
#pragma once
#include "../ps_errors.hpp"
