// eval.hpp — drop-in name for the reference header proj/include/planestereo/eval.hpp;
// of it this build provides accuracy() (GPU), declared in planestereo.hpp.
#pragma once
#include "planestereo/planestereo.hpp"
