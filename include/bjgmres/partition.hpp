// Forwarding header: keeps the reference's #include "bjgmres/partition.hpp"
// (proj/include/bjgmres/partition.hpp) valid; everything lives in bjgmres_b200.hpp.
#pragma once
#include "../bjgmres_b200.hpp"
