#!/usr/bin/env python
"""theta_m for the truncated Taylor exponential (engine.cpp expm_taylor): the largest ||X||_1 with
sum_k |c_k| ||X||^(k-1) <= 2^-53, c_k the series of h_m(X) = log(e^-X T_m(X)) (relative backward
error bound), computed in exact rational arithmetic."""
from fractions import Fraction as F
import math
def series_exp(n, sign=1):
    c=[F(0)]*n; f=F(1)
    for k in range(n):
        c[k]=F(sign)**k/math.factorial(k)
    return c
def mul(a,b,n):
    r=[F(0)]*n
    for i,x in enumerate(a[:n]):
        if x==0: continue
        for j,y in enumerate(b[:n-i]):
            r[i+j]+=x*y
    return r
def log1p_series(a,n):  # log(1+a), a has zero constant term
    r=[F(0)]*n; p=[F(1)]+[F(0)]*(n-1)
    for k in range(1,n):
        p=mul(p,a,n)
        if all(v==0 for v in p): break
        s=F((-1)**(k+1),k)
        r=[x+s*y for x,y in zip(r,p)]
    return r
u=2.0**-53
for m in [12,14,16,18,20,24,28,32]:
    n=m+1+60
    Tm=[F(1,math.factorial(k)) if k<=m else F(0) for k in range(n)]
    e=series_exp(n,-1)
    prod=mul(e,Tm,n); prod[0]-=1
    h=log1p_series(prod,n)
    c=[abs(float(x)) for x in h]
    f=lambda t: sum(c[k]*t**(k-1) for k in range(1,n))
    lo,hi=0.0,20.0
    for _ in range(200):
        mid=(lo+hi)/2
        if f(mid)<=u: lo=mid
        else: hi=mid
    print(m, lo)
