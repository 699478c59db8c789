// Forwarding header: keeps the reference's #include "bjgmres/preconditioner.hpp"
// (proj/include/bjgmres/preconditioner.hpp) valid; everything lives in bjgmres_b200.hpp.
#pragma once
#include "../bjgmres_b200.hpp"
