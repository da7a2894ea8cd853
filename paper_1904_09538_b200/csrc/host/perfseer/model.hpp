// Reference-compatible include path (perfseer/model.hpp) for code written
// against the reference API; the declarations live in ps_model.hpp.
#pragma once
#include "../ps_model.hpp"
