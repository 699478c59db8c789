// Forwarding header: keeps the reference's #include "bjgmres/gmres.hpp"
// (proj/include/bjgmres/gmres.hpp) valid; everything lives in bjgmres_b200.hpp.
#pragma once
#include "../bjgmres_b200.hpp"
