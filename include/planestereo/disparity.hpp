// disparity.hpp — drop-in name for the reference header proj/include/planestereo/disparity.hpp;
// the whole API is declared in planestereo.hpp.
#pragma once
#include "planestereo/planestereo.hpp"
