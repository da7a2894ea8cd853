// Reference-compatible include path (perfseer/oracle.hpp) for code written
// against the reference API; the declarations live in ps_enumerate.hpp.
#pragma once
#include "../ps_enumerate.hpp"
