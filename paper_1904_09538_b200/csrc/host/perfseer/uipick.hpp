// Reference-compatible include path (perfseer/uipick.hpp) for code written
// against the reference API; the declarations live in ps_catalog.hpp.
#pragma once
#include "../ps_catalog.hpp"
