// Forwarding header: keeps the reference's #include "bjgmres/lu.hpp"
// (proj/include/bjgmres/lu.hpp) valid; everything lives in bjgmres_b200.hpp.
#pragma once
#include "../bjgmres_b200.hpp"
