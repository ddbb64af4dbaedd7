// Forwarding header: the reference's blco/cpals.hpp, served by the B200 build.
#pragma once
#include "blco/b200.hpp"
