// Coefficients of the product-saving Taylor schemes for the propagator R(A) = y(A/2^s)^(2^s)
// (derived by tools/derive_expm_schemes.py in 50-digit arithmetic; tests/test_schemes.py
// checks that every set reproduces the Taylor coefficients of exp).  Shared by tiny.cuh and
// large.cu.
//
// s4 -- degree 12 in 4 products (theta_12 = 0.3352):
//   A2 = A A, A3 = A2 A,  Z = (X4 A + X5 A2 + X6 A3) A3 + Z0 I + Z1 A + Z2 A2 + Z3 A3,
//   y = (Z + B0 I + B1 A + B2 A2 + B3 A3) Z + C0 I + C1 A + C2 A2 + C3 A3
// s5 -- degree 18 in 5 products (theta_18 = 1.1433):
//   A2 = A A, A3 = A2 A, A6 = A3 A3,  P = A + BE2 A2 + BE3 A3,  Q = GA2 A2 + GA3 A3 + GA6 A6,
//   Z = P Q,  y = (Z + b(A)) (Z + e(A)) + c(A),   b, e, c on the basis I, A, A2, A3, A6
#pragma once

#define SQOC_S4_Z0 0.0
#define SQOC_S4_Z1 2.1763083362520447e-12
#define SQOC_S4_Z2 0.11462406647905307
#define SQOC_S4_Z3 0.012167782611650191
#define SQOC_S4_X4 2.1931723165325633e-3
#define SQOC_S4_X5 2.7414653956657041e-4
#define SQOC_S4_X6 4.5691089927761735e-5
#define SQOC_S4_B0 5.5174437753427168
#define SQOC_S4_B1 1.3093238729655877
#define SQOC_S4_B2 4.3247187526118505e-3
#define SQOC_S4_B3 9.6586056829543493e-3
#define SQOC_S4_C0 1.0
#define SQOC_S4_C1 0.99999999998799234
#define SQOC_S4_C2 -0.13243184210217061
#define SQOC_S4_C3 -0.050548416421633109

#define SQOC_S5_BE2 0.08
#define SQOC_S5_BE3 8.8888888888888889e-3
#define SQOC_S5_GA2 9.2674026525459185e-3
#define SQOC_S5_GA3 1.6998410509078933e-3
#define SQOC_S5_GA6 1.4059892894192666e-6
#define SQOC_S5_B0 0.0
#define SQOC_S5_B1 -0.067640451907138191
#define SQOC_S5_B2 0.067596130177045965
#define SQOC_S5_B3 0.029555257042931553
#define SQOC_S5_B6 -1.391802575160607e-5
#define SQOC_S5_E0 -11.148502971774368
#define SQOC_S5_E1 1.6125176868819238
#define SQOC_S5_E2 0.12477411482493252
#define SQOC_S5_E3 0.022573155818051032
#define SQOC_S5_E6 1.9579475957000984e-5
#define SQOC_S5_C0 1.0
#define SQOC_S5_C1 0.24591022090110864
#define SQOC_S5_C2 1.3626670832081905
#define SQOC_S5_C3 0.49892102569169427
#define SQOC_S5_C6 -6.4092743005853664e-4
